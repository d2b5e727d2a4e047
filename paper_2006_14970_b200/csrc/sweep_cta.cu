// K3s: the band-CTA variant of the big-level sweep (the dependency structure,
// boundary streams, rings and output path are those of sweep.cu; read that
// first).  One CTA per band: warps 0-2 run the F_c / B_c recurrence of channel
// c = warp, warp 3 computes the band's alpha-only coefficients (the 2x2 system
// of multilevel.cpp:94-118 is common to the three channels, multilevel.hpp:
// 37-43) once per pixel and sweep and hands them to the channel warps through
// a double-buffered shared-memory record, two steps at a time:
//
//   coefficient warp  P(0) | P(1) P(2) | P(3) P(4) | ...
//   channel warps          | C(0) C(1) | C(2) C(3) | ...      (C(j) reads P(j))
//                        sync       sync sync
//
// P(j) writes the records of steps 2j, 2j+1 into buffer j&1 while the channel
// warps consume buffer (j-1)&1; a CTA barrier after each half-group orders
// them.  Per channel warp this replaces the ~27 instructions of the
// coefficient algebra and 5 alpha loads per pixel with 3 shared loads and 2
// multiplies (p*I_c, q*I_c); the alpha ring exists once per band.  The
// results are bitwise those of sweep.cu (same operations, same order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "fgm_device.cuh"
#include "fgm_internal.h"

namespace fgm {
namespace {

__device__ __forceinline__ void cp_async16(unsigned sdst, const float* gsrc, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16_if(unsigned sdst, const float* gsrc, unsigned pred) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16;\n}" ::"r"(sdst),
        "l"(gsrc), "r"(pred)
        : "memory");
}
__device__ __forceinline__ void cp_async4(unsigned sdst, const float* gsrc, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sdst), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ float4 ld_relaxed_v4(const float* p) {
    float4 v;
    asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_v4(float* p, float4 v) {
    asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
}
__device__ __forceinline__ void st_relaxed_v2(float* p, float2 v) {
    asm volatile("st.relaxed.gpu.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y));
}
extern __shared__ float4 cta_sm4[];
__device__ __forceinline__ float* smf() { return reinterpret_cast<float*>(cta_sm4); }
__device__ __forceinline__ float lds(int i) { return smf()[i]; }
__device__ __forceinline__ float4 lds4(int i) { return reinterpret_cast<const float4*>(smf() + i)[0]; }
__device__ __forceinline__ void sts(int i, float v) { smf()[i] = v; }
__device__ __forceinline__ void sts4(int i, float4 v) { reinterpret_cast<float4*>(smf() + i)[0] = v; }
__device__ __forceinline__ void stg(float* p, float v) { __stcg(p, v); }
__device__ __forceinline__ bool is_sentinel(float v) { return __float_as_uint(v) == kStreamSentinel; }
__device__ __forceinline__ constexpr int orow(int j) { return j + (j >> 4); }

// Shared memory of one band CTA, in floats: the coefficient warp's alpha ring,
// the record buffers, then one region per channel warp (image ring, F/B rings,
// output ring, chunk buffer).  Ring geometry and load leads as in sweep.cu.
template <int K>
struct GeomS {
    static constexpr int RW = 32, SH = K - 1, MIR = K <= 2 ? 4 : 8, RS = RW + MIR;
    static constexpr int M = 4;
    static constexpr int L = 4 * M + 1;   // channel warps' lead (image W1 = 1, F/B W1 = 1; as sweep.cu)
    static constexpr int LP = 4 * M + 2;  // coefficient warp's lead: it runs one half-group ahead (W1 = 3)
    static constexpr int NA = 33 + K, NI = 31 + K, NF = 33, OW = 16, OPL = 33 * OW;
    static constexpr int CK = kChunk;
    static constexpr int NS = 2 * K;  // records per half-group: 2 steps x K slots
    static constexpr int OFF_A = 0;
    static constexpr int OFF_R0 = OFF_A + NA * RS;          // [2][NS][32] float4: dL dR dU dD
    static constexpr int OFF_R1 = OFF_R0 + 2 * NS * 32 * 4;  // [2][NS][32] float4: A A2 Bc p
    static constexpr int OFF_R2 = OFF_R1 + 2 * NS * 32 * 4;  // [2][NS][32] float: q
    static constexpr int OFF_CH = OFF_R2 + 2 * NS * 32;
    static constexpr int C_I = 0, C_F = C_I + NI * RS, C_B = C_F + NF * RS, C_O = C_B + NF * RS;
    static constexpr int C_C = C_O + 2 * OPL;
    static constexpr int CH = CK * K * 2, CH4 = CH / 4;
    static constexpr int PC = (C_C + CH + 3) / 4 * 4;  // one channel region
    static constexpr int TOTAL = OFF_CH + 3 * PC;
    static_assert(LP + (2 * K - 2) + 4 <= RW && L + (2 * K - 2) + 4 <= RW, "ring too small for its lead");
    static_assert(2 + SH <= MIR && RS % 4 == 0 && OFF_CH % 4 == 0, "layout");
    static_assert(CH4 <= 32, "a chunk is at most one float4 per lane");
};

// One global row of up to 4 planes streamed into rings whose row addresses
// are held explicitly (s[p]); vm masks the planes the lane streams.
struct RowSrcS {
    const float* g[4];
    unsigned s[4];
    unsigned vm;
    int r;
};

template <int K, bool V4>
__device__ __forceinline__ void put_blocks(const RowSrcS& rs, int x0, int w) {
    using G = GeomS<K>;
    if (x0 < 0 || x0 >= w) return;
    const int nb = min(w - x0, 4) * 4;
    const int c = x0 & (G::RW - 1);
    const bool mir = c < G::MIR;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        if (!(rs.vm & (1u << p))) continue;
        const float* g = rs.g[p] + x0;
        const unsigned d = rs.s[p] + 4u * c;
        if (V4) {
            cp_async16(d, g, nb);
            if (mir) cp_async16(d + 4u * G::RW, g, nb);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int ok = 4 * i < nb;
                cp_async4(d + 4 * i, ok ? g + i : g, ok ? 4 : 0);
                if (mir) cp_async4(d + 4u * G::RW + 4 * i, ok ? g + i : g, ok ? 4 : 0);
            }
        }
    }
}

template <int K>
__device__ __forceinline__ void put_blocks_fast(const RowSrcS& rs, int x0) {  // x0 in [0, w-4]
    using G = GeomS<K>;
    const unsigned c = unsigned(x0) & (G::RW - 1);
    const unsigned mir = c < unsigned(G::MIR) ? 1u : 0u;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float* g = rs.g[p] + unsigned(x0);
        const unsigned d = rs.s[p] + 4u * c;
        const unsigned on = (rs.vm >> p) & 1u;
        cp_async16_if(d, g, on);
        cp_async16_if(d + 4u * G::RW, g, on & mir);
    }
}

// ---------------------------------------------------------------------------
// Coefficient warp
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ RowSrcS alpha_row(const SweepJob& J, int y0, int r, bool on, unsigned sbase) {
    using G = GeomS<K>;
    RowSrcS rs{};
    const int y = y0 + r;
    const bool ok = on && y >= 0 && y < J.h;
    rs.g[0] = rs.g[1] = rs.g[2] = rs.g[3] = J.alpha + (long long)(ok ? y : 0) * J.ipitch;
    rs.s[0] = rs.s[1] = rs.s[2] = rs.s[3] = sbase + 4u * unsigned(G::OFF_A + max(r + K, 0) * G::RS);
    rs.vm = ok ? 1u : 0u;
    rs.r = r;
    return rs;
}

// Records of the half-group hh (steps 2hh, 2hh+1) into buffer hh & 1.  The
// pixel of slot k at step tt is (tt - lane - k, y0 + lane - k); its alpha
// neighbourhood is read around base step tt - 1 exactly as sweep.cu's
// next_coef.  G: clamp neighbours at the image border.
template <int K, bool G>
__device__ __forceinline__ void produce(int hh, int lane, int y0, int w, int h, float eps, float omega) {
    using Gm = GeomS<K>;
    const int buf = hh & 1;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const int tt = 2 * hh + s;
        const int rc = Gm::OFF_A + lane * Gm::RS + ((tt - 1 - lane - Gm::SH) & (Gm::RW - 1));
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int dp = 1 - k + Gm::SH, ar = K - k;
            const int i0 = rc + ar * Gm::RS + dp;
            const float a = lds(i0);
            float aL = lds(i0 - 1), aR = lds(i0 + 1), aU = lds(i0 - Gm::RS), aD = lds(i0 + Gm::RS);
            if (G) {
                const int x = tt - lane - k, y = y0 + lane - k;
                if (x <= 0) aL = a;
                if (x >= w - 1) aR = a;
                if (y <= 0) aU = a;
                if (y >= h - 1) aD = a;
            }
            // pixel_coef1 (fgm_device.cuh) without the image factor
            const float dL = edge_weight(a, aL, eps, omega), dR = edge_weight(a, aR, eps, omega);
            const float dU = edge_weight(a, aU, eps, omega), dD = edge_weight(a, aD, eps, omega);
            const float S = __fadd_rn(__fadd_rn(__fadd_rn(dL, dR), dU), dD);
            const float u0 = a, u1 = __fsub_rn(1.0f, a);
            const float u00 = __fmul_rn(u0, u0), u11 = __fmul_rn(u1, u1), u01 = __fmul_rn(u0, u1);
            const float iS = rcp_approx(S);
            const float iD = rcp_approx(__fadd_rn(__fadd_rn(u00, u11), S));
            const float A = __fmul_rn(iD, __fmaf_rn(u11, iS, 1.0f));
            const float A2 = __fmul_rn(iD, __fmaf_rn(u00, iS, 1.0f));
            const float Bc = -__fmul_rn(iD, __fmul_rn(u01, iS));
            const int idx = (buf * Gm::NS + s * K + k) * 32 + lane;
            sts4(Gm::OFF_R0 + 4 * idx, make_float4(dL, dR, dU, dD));
            sts4(Gm::OFF_R1 + 4 * idx, make_float4(A, A2, Bc, __fmul_rn(iD, u0)));
            sts(Gm::OFF_R2 + idx, __fmul_rn(iD, u1));
        }
    }
}

template <int K, bool V4>
__device__ __forceinline__ void run_producer(const SweepJob& J, int q, int lane, unsigned sbase, float eps,
                                             float omega) {
    using Gm = GeomS<K>;
    const int w = J.w, h = J.h, y0 = q * kBandRows;
    const int Umax = w + K - 1, tend = 31 + Umax;
    const RowSrcS own = alpha_row<K>(J, y0, lane, true, sbase);
    const bool has_x = lane >= 32 - K || lane == 0;
    const RowSrcS ext = alpha_row<K>(J, y0, lane == 0 ? 32 : lane - 32, has_x, sbase);
    // everything "issued before group 0", complete before the first records
    const int lo = (Gm::LP - own.r) & ~3, le = (Gm::LP - ext.r) & ~3;
    for (int x0 = 0; x0 <= lo; x0 += 4) put_blocks<K, V4>(own, x0, w);
    for (int x0 = 0; x0 <= le; x0 += 4) put_blocks<K, V4>(ext, x0, w);
    cp_commit();
    cp_wait<0>();
    __syncwarp();
    const bool yband = y0 - (K - 1) <= 0 || y0 + 31 >= h - 1;
    auto prod = [&](int hh) {
        if (!yband && 2 * hh >= 32 + K && 2 * hh + 2 <= w - 2)
            produce<K, false>(hh, lane, y0, w, h, eps, omega);
        else
            produce<K, true>(hh, lane, y0, w, h, eps, omega);
    };
    prod(0);
    __syncthreads();
    const int issue_lo = 32 + 3 - 4 - Gm::LP, issue_hi = w - 4 - 4 - Gm::LP - K;
    for (int t4 = 0; t4 < tend; t4 += 4) {
        cp_wait<Gm::M - 1>();
        __syncwarp();
        prod(t4 / 2 + 1);
        __syncthreads();
        prod(t4 / 2 + 2);
        __syncthreads();
        // (the slots the next blocks overwrite are older than every read of
        // the next group: the span static_assert)
        if (V4 && !yband && t4 >= issue_lo && t4 < issue_hi) {
            put_blocks_fast<K>(own, (t4 + 4 + Gm::LP - own.r) & ~3);
            put_blocks_fast<K>(ext, (t4 + 4 + Gm::LP - ext.r) & ~3);
        } else {
            put_blocks<K, V4>(own, (t4 + 4 + Gm::LP - own.r) & ~3, w);
            if (has_x) put_blocks<K, V4>(ext, (t4 + 4 + Gm::LP - ext.r) & ~3, w);
        }
        cp_commit();
    }
    cp_wait<0>();
}

// ---------------------------------------------------------------------------
// Channel warps
// ---------------------------------------------------------------------------
template <int K>
struct ChCtx {
    int base;  // float offset of this channel's region
    int lb;    // base + lane * RS
    int ob;    // output ring row orow(lane)
    int lane, y0, w, h;
    bool has_up, has_down;
    int Umax;
    float* my_stream;
    float* FO;
    float* BO;
    int opitch;
};

template <int K>
struct ChState {
    float2 outp[K];
    float2 rprev[K];
};

template <int K, bool G>
__device__ __forceinline__ void chan_step(ChState<K>& st, const ChCtx<K>& x_, int tr, int buf, int s) {
    using Gm = GeomS<K>;
    constexpr int OW = Gm::OW;
    const int lane = x_.lane, y0 = x_.y0, w = x_.w, h = x_.h;
    const int c = (tr - lane - Gm::SH) & (Gm::RW - 1);
    const int rc = x_.lb + c;

    float2 recv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        recv[k].x = __shfl_up_sync(kFull, st.outp[k].x, 1);
        recv[k].y = __shfl_up_sync(kFull, st.outp[k].y, 1);
    }
    if (lane == 0 && x_.has_up && (!G || (tr >= 0 && tr < x_.Umax))) {
        const int cn = x_.base + Gm::C_C + (tr % Gm::CK) * K * 2;
#pragma unroll
        for (int k = 0; k < K; ++k) recv[k] = make_float2(lds(cn + 2 * k), lds(cn + 2 * k + 1));
    }

    float2 nv[K];
    const int xs0 = tr - lane;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        // this step's record of slot k, completed with the channel's image term
        const int idx = (buf * Gm::NS + s * K + k) * 32 + lane;
        const float4 r0 = lds4(Gm::OFF_R0 + 4 * idx), r1 = lds4(Gm::OFF_R1 + 4 * idx);
        const float qq = lds(Gm::OFF_R2 + idx);
        const float I = lds(rc + Gm::C_I + (K - 1 - k) * Gm::RS + (Gm::SH - k));
        Coef1 co;
        co.dL = r0.x;
        co.dR = r0.y;
        co.dU = r0.z;
        co.dD = r0.w;
        co.A = r1.x;
        co.A2 = r1.y;
        co.Bc = r1.z;
        co.pI = __fmul_rn(r1.w, I);
        co.qI = __fmul_rn(qq, I);
        float2 L = st.outp[k], U = recv[k], R, D;
        if (k == 0) {
            R = make_float2(lds(rc + Gm::C_F + 1 + Gm::SH), lds(rc + Gm::C_B + 1 + Gm::SH));
            D = make_float2(lds(rc + Gm::C_F + Gm::RS + Gm::SH), lds(rc + Gm::C_B + Gm::RS + Gm::SH));
        } else {
            R = recv[k - 1];
            D = st.outp[k - 1];
        }
        if (G) {
            const int x = xs0 - k, y = y0 + lane - k;
            const float2 self = k == 0 ? make_float2(lds(rc + Gm::C_F + Gm::SH), lds(rc + Gm::C_B + Gm::SH))
                                       : st.rprev[k > 0 ? k - 1 : 0];
            if (!(x > 0)) L = self;
            if (!(x < w - 1)) R = self;
            if (!(y > 0)) U = self;
            if (!(y < h - 1)) D = self;
        }
        nv[k] = pixel_apply1(co, L, R, U, D);
    }

    {  // output ring (last sweep only)
        bool ok = true;
        if (G) {
            const int x = xs0 - (K - 1);
            ok = x >= 0 && x < w && y0 + lane - (K - 1) >= 0 && y0 + lane - (K - 1) < h;
        }
        if (ok) {
            const int o = x_.ob + (c & (OW - 1));
            sts(o, nv[K - 1].x);
            sts(o + Gm::OPL, nv[K - 1].y);
        }
    }

    if (x_.has_down && lane == kBandRows - 1 && (!G || (tr - 31 >= 0 && tr - 31 < x_.Umax))) {
        float* dst = x_.my_stream + size_t(tr - 31) * K * 2;
        if (K % 2 == 0) {
#pragma unroll
            for (int k = 0; k + 1 < K; k += 2)
                st_relaxed_v4(dst + 2 * k, make_float4(nv[k].x, nv[k].y, nv[k + 1].x, nv[k + 1].y));
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) st_relaxed_v2(dst + 2 * k, nv[k]);
        }
    }

    __syncwarp();
    {  // flush completed 16-column output row segments (as sweep.cu)
        const int col = lane & (OW - 1);
        const int u = tr - (K - 1) - (OW - 1);
        const int jf = (u & (OW - 1)) + (lane & 16);
        const int xs = (u & ~(OW - 1)) - (lane & 16);
        bool ok = true;
        if (G) {
            const int yf = y0 + jf - (K - 1);
            ok = xs >= 0 && xs + OW - 1 < w && yf >= 0 && yf < h;
        }
        if (ok) {
            const unsigned off = unsigned(jf * x_.opitch + xs + col);
            const int o = x_.base + Gm::C_O + orow(jf) * OW + col;
            stg(x_.FO + off, lds(o));
            stg(x_.BO + off, lds(o + Gm::OPL));
        }
        if (G && ((w - 1) & (OW - 1)) != OW - 1) {
            const int je = tr - (K - 1) - (w - 1);
            const int x0 = (w - 1) & ~(OW - 1);
            const int ye = y0 + je - (K - 1);
            if (je >= 0 && je < 32 && ye >= 0 && ye < h && lane < w - x0) {
                const unsigned off = unsigned(je * x_.opitch + x0 + lane);
                const int o = x_.base + Gm::C_O + orow(je) * OW + lane;
                stg(x_.FO + off, lds(o));
                stg(x_.BO + off, lds(o + Gm::OPL));
            }
        }
    }

#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (G) st.rprev[k] = recv[k];
        st.outp[k] = nv[k];
    }
}

template <int K>
__device__ __forceinline__ bool chunk_complete(float4 q, int u0, int Umax, int lane) {
    using G = GeomS<K>;
    const int nvalid = min(G::CK, Umax - u0) * K * 2;
    const bool mine = lane < G::CH4 && 4 * lane < nvalid;
    if (!mine) return true;
    const int b = 4 * lane;
    return !(is_sentinel(q.x) || (b + 1 < nvalid && is_sentinel(q.y)) || (b + 2 < nvalid && is_sentinel(q.z)) ||
             (b + 3 < nvalid && is_sentinel(q.w)));
}

template <int K>
__device__ __forceinline__ void acquire_chunk(float4 v, const float* up_stream, int u0, int Umax, int lane,
                                              int chunk) {
    using G = GeomS<K>;
    const int nvalid = min(G::CK, Umax - u0) * K * 2;
    const bool mine = lane < G::CH4 && 4 * lane < nvalid;
    while (!__all_sync(kFull, chunk_complete<K>(v, u0, Umax, lane))) {
        __nanosleep(32);
        if (mine) v = ld_relaxed_v4(up_stream + size_t(u0) * K * 2 + 4 * lane);
    }
    if (mine) sts4(chunk + 4 * lane, v);
}

template <int K>
__device__ __forceinline__ RowSrcS chan_row(const SweepJob& J, int ch, int y0, int r, bool doI, bool doF, int base,
                                            unsigned sbase) {
    using G = GeomS<K>;
    RowSrcS rs{};
    const int y = y0 + r;
    const bool ok = y >= 0 && y < J.h;
    const long long oi = (long long)(ok ? y : 0) * J.ipitch, of = (long long)(ok ? y : 0) * J.fpitch;
    rs.g[0] = rs.g[1] = J.img + ch * J.istride + oi;
    rs.g[2] = J.fg_in + ch * J.fstride + of;
    rs.g[3] = J.bg_in + ch * J.fstride + of;
    const unsigned b = sbase + 4u * unsigned(base);
    rs.s[0] = rs.s[1] = b + 4u * unsigned(G::C_I + max(r + K - 1, 0) * G::RS);
    rs.s[2] = b + 4u * unsigned(G::C_F + max(r, 0) * G::RS);
    rs.s[3] = b + 4u * unsigned(G::C_B + max(r, 0) * G::RS);
    rs.vm = ok ? (doI ? 2u : 0u) | (doF ? 12u : 0u) : 0u;
    rs.r = r;
    return rs;
}

template <int K, bool V4>
__device__ __forceinline__ void run_channel(const SweepJob& J, int q, int ch, int lane, unsigned sbase) {
    using Gm = GeomS<K>;
    const int w = J.w, h = J.h, y0 = q * kBandRows;
    const int Umax = w + K - 1, tend = 31 + Umax;
    const size_t slen = sweep_stream_len(w, K);
    const int sid = q * 3 + ch;
    const float* up_stream = q > 0 ? J.stream + size_t(sid - 3) * slen : nullptr;

    ChCtx<K> cx;
    cx.base = Gm::OFF_CH + ch * Gm::PC;
    cx.lb = cx.base + lane * Gm::RS;
    cx.ob = cx.base + Gm::C_O + orow(lane) * Gm::OW;
    cx.lane = lane;
    cx.y0 = y0;
    cx.w = w;
    cx.h = h;
    cx.has_up = q > 0;
    cx.has_down = q < J.nb - 1;
    cx.Umax = Umax;
    cx.my_stream = J.stream + size_t(sid) * slen;
    cx.FO = J.fg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    cx.BO = J.bg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    cx.opitch = J.opitch;

    const RowSrcS own = chan_row<K>(J, ch, y0, lane, true, true, cx.base, sbase);
    const bool has_x = lane >= 33 - K || lane == 0;
    const RowSrcS ext = chan_row<K>(J, ch, y0, lane == 0 ? 32 : lane - 32, lane >= 33 - K, lane == 0, cx.base, sbase);

    ChState<K> st;
#pragma unroll
    for (int k = 0; k < K; ++k) st.outp[k] = st.rprev[k] = make_float2(0.0f, 0.0f);

    constexpr int t0 = -4;  // loads "issued before group 0" = sweep.cu's prologue
    {
        const int lo = (t0 + Gm::L - own.r) & ~3, le = (t0 + Gm::L - ext.r) & ~3;
        for (int x0 = 0; x0 <= lo; x0 += 4) put_blocks<K, V4>(own, x0, w);
        if (has_x)
            for (int x0 = 0; x0 <= le; x0 += 4) put_blocks<K, V4>(ext, x0, w);
        // sweep.cu also issues group -4's blocks at the end of its init group
        put_blocks<K, V4>(own, (t0 + 4 + Gm::L - own.r) & ~3, w);
        if (has_x) put_blocks<K, V4>(ext, (t0 + 4 + Gm::L - ext.r) & ~3, w);
    }
    cp_commit();
#pragma unroll
    for (int i = 1; i < Gm::M; ++i) cp_commit();
    float4 pend = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool lane_ch = lane < Gm::CH4;
    bool pend_ok = false;
    if (cx.has_up && lane_ch) pend = ld_relaxed_v4(up_stream + 4 * lane);
    __syncthreads();  // the first half-group's records

    const bool yband = y0 - (K - 1) <= 0 || y0 + 31 >= h - 1;
    const int fast_lo = 32 + K, fast_hi = w - 2;
    const int issue_lo = 32 + 3 - 4 - Gm::L, issue_hi = w - 4 - 4 - Gm::L - K;
    for (int t4 = 0; t4 < tend; t4 += 4) {
        cp_wait<Gm::M - 1>();
        __syncwarp();
        if (cx.has_up && t4 < Umax) {
            const int nxt = (t4 & ~(Gm::CK - 1)) + Gm::CK;
            if ((t4 % Gm::CK) == 0) {
                acquire_chunk<K>(pend, up_stream, t4, Umax, lane, cx.base + Gm::C_C);
                pend_ok = false;
                if (nxt < Umax && lane_ch) pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
            } else if (!pend_ok && nxt < Umax) {
                pend_ok = __all_sync(kFull, chunk_complete<K>(pend, nxt, Umax, lane));
                if (!pend_ok && lane_ch) pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
            }
        }
        __syncwarp();
        const bool fast = !yband && t4 >= fast_lo && t4 + 4 <= fast_hi;
        const int hb = (t4 / 2) & 1;  // buffer of the first half-group
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            if (fast) {
                chan_step<K, false>(st, cx, t4 + 2 * half, hb ^ half, 0);
                chan_step<K, false>(st, cx, t4 + 2 * half + 1, hb ^ half, 1);
            } else {
                chan_step<K, true>(st, cx, t4 + 2 * half, hb ^ half, 0);
                chan_step<K, true>(st, cx, t4 + 2 * half + 1, hb ^ half, 1);
            }
            __syncthreads();
        }
        if (V4 && !yband && t4 >= issue_lo && t4 < issue_hi) {
            put_blocks_fast<K>(own, (t4 + 4 + Gm::L - own.r) & ~3);
            RowSrcS e = ext;
            if (!has_x) e.vm = 0;
            put_blocks_fast<K>(e, (t4 + 4 + Gm::L - ext.r) & ~3);
        } else {
            put_blocks<K, V4>(own, (t4 + 4 + Gm::L - own.r) & ~3, w);
            if (has_x) put_blocks<K, V4>(ext, (t4 + 4 + Gm::L - ext.r) & ~3, w);
        }
        cp_commit();
    }
    cp_wait<0>();
}

template <int K, bool V4>
__global__ void __launch_bounds__(128) sweep_cta_kernel(const SweepJob* __restrict__ jobs,
                                                        const int2* __restrict__ order, int total_items,
                                                        unsigned* ticket, float eps, float omega) {
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(cta_sm4));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ unsigned s_tk;
    for (;;) {
        __syncthreads();  // the previous band is done with the shared memory
        if (threadIdx.x == 0) s_tk = atomicAdd(ticket, 1u);
        __syncthreads();
        const unsigned tk = s_tk;
        if (tk >= unsigned(total_items)) return;
        const int2 jb = order[tk];  // (job, band)
        const SweepJob J = jobs[jb.x];
        const bool v4 = V4 && J.vec4;
        if (warp == 3) {
            if (v4)
                run_producer<K, V4>(J, jb.y, lane, sbase, eps, omega);
            else
                run_producer<K, false>(J, jb.y, lane, sbase, eps, omega);
        } else {
            if (v4)
                run_channel<K, V4>(J, jb.y, warp, lane, sbase);
            else
                run_channel<K, false>(J, jb.y, warp, lane, sbase);
        }
    }
}

template <int K>
cudaError_t launch_k(const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket, float eps,
                     float omega, cudaStream_t s) {
    static int grid_cap = 0;
    constexpr size_t smem = size_t(GeomS<K>::TOTAL) * sizeof(float);
    if (grid_cap == 0) {
        cudaError_t e = cudaFuncSetAttribute(sweep_cta_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_cta_kernel<K, true>, 128, smem);
        grid_cap = std::max(1, sms * std::max(1, per_sm));
    }
    const int grid = std::max(1, std::min(total_items, grid_cap));
    sweep_cta_kernel<K, true><<<grid, 128, smem, s>>>(jobs_dev, order_dev, total_items, ticket, eps, omega);
    return cudaGetLastError();
}

}  // namespace

int sweep_cta_supported_k(int K) { return K >= 1 && K <= 2; }

cudaError_t launch_sweep_cta(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_bands,
                             unsigned* ticket, float eps, float omega, cudaStream_t s) {
    switch (K) {
        case 1: return launch_k<1>(jobs_dev, order_dev, total_bands, ticket, eps, omega, s);
        case 2: return launch_k<2>(jobs_dev, order_dev, total_bands, ticket, eps, omega, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fgm
