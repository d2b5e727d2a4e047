// K3f: the throughput variant of the big-level sweep (see sweep.cu for the
// dependency structure, which is identical).  One warp per band handles all
// three colour channels, and each pixel's alpha-only coefficients are computed
// exactly once: by slot 0 (the first fused sweep), one step ahead, and handed
// to slot k at lane j+1 two steps later (the same pixel in skewed
// coordinates) by shfl.up -- lane 0 gets them from the band above through the
// boundary stream.  Per pixel-update this needs ~2.5x fewer instructions than
// the per-(band, channel) kernel, which in turn has 3x more warps per band;
// the solver picks this kernel when a launch has enough bands to fill the GPU
// (batches, 16k images) and the other one for latency-bound single images.
//
// Stream entry per skewed column u (EW floats, 16-byte padded):
//   [0, FBW)      K x 3 (F_c, B_c) of the band's last row at column u
//   [FBW, EW)     the (K-1) passed coefficient sets (13 floats each) that the
//                 last row used at column u-1 (written one column ahead)
// Every stored float is an arithmetic result (saturated outputs or products),
// so it can never equal the NaN sentinel the buffer is filled with.
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
                 "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ bool is_sentinel(float v) { return __float_as_uint(v) == kStreamSentinel; }

// The coefficient set handed from slot k to slot k+1 (Coef3 + the per-channel
// image terms p*I_c, q*I_c).
struct PassC {
    float dL, dR, dU, dD, A, A2, Bn, pI[3], qI[3];  // Bn = -Bc > 0
};
constexpr int kPassFloats = 13;

__device__ __forceinline__ float pc_get(const PassC& p, int i) {
    switch (i) {
        case 0: return p.dL;
        case 1: return p.dR;
        case 2: return p.dU;
        case 3: return p.dD;
        case 4: return p.A;
        case 5: return p.A2;
        case 6: return p.Bn;
        case 7: return p.pI[0];
        case 8: return p.pI[1];
        case 9: return p.pI[2];
        case 10: return p.qI[0];
        case 11: return p.qI[1];
        default: return p.qI[2];
    }
}
__device__ __forceinline__ void pc_set(PassC& p, int i, float v) {
    switch (i) {
        case 0: p.dL = v; break;
        case 1: p.dR = v; break;
        case 2: p.dU = v; break;
        case 3: p.dD = v; break;
        case 4: p.A = v; break;
        case 5: p.A2 = v; break;
        case 6: p.Bn = v; break;
        case 7: p.pI[0] = v; break;
        case 8: p.pI[1] = v; break;
        case 9: p.pI[2] = v; break;
        case 10: p.qI[0] = v; break;
        case 11: p.qI[1] = v; break;
        default: p.qI[2] = v; break;
    }
}

__device__ __forceinline__ float2 apply_c(const PassC& co, int c, float2 L, float2 R, float2 U, float2 D) {
    float SF = __fmul_rn(co.dL, L.x);
    float SB = __fmul_rn(co.dL, L.y);
    SF = __fmaf_rn(co.dD, D.x, SF);
    SB = __fmaf_rn(co.dD, D.y, SB);
    SF = __fmaf_rn(co.dR, R.x, SF);
    SB = __fmaf_rn(co.dR, R.y, SB);
    SF = __fmaf_rn(co.dU, U.x, SF);
    SB = __fmaf_rn(co.dU, U.y, SB);
    return make_float2(__saturatef(__fmaf_rn(co.A, SF, __fmaf_rn(-co.Bn, SB, co.pI[c]))),
                       __saturatef(__fmaf_rn(co.A2, SB, __fmaf_rn(-co.Bn, SF, co.qI[c]))));
}

template <int K>
struct GeomF {
    static constexpr int kLeadA = 20;  // alpha ring lead (columns), 32-wide ring
    static constexpr int kLeadF = 8;   // image and F/B ring lead, 16-wide rings
    static constexpr int NA = 34;      // alpha rows -1 .. 32
    static constexpr int IR = 33;      // image rows 0 .. 31, padded: irow(r) = r + r/16
    static constexpr int FR = 35;      // F/B rows 0 .. 32, padded: frow(r) = r + r/16
    static constexpr int OW = 8;       // output ring columns
    static constexpr int OR = 35;      // output rows, padded: orow(j) = j + j/8
    static constexpr int OFF_A = 0;
    static constexpr int OFF_I = OFF_A + NA * 32;
    static constexpr int OFF_F = OFF_I + 3 * IR * 16;
    static constexpr int OFF_O = OFF_F + 6 * FR * 16;
    static constexpr int OFF_C = OFF_O + 6 * OR * OW;
    static constexpr int FBW = (6 * K + 3) / 4 * 4;
    static constexpr int CW = (kPassFloats * (K - 1) + 3) / 4 * 4;
    static constexpr int EW = FBW + CW;
    static constexpr int CH = kChunk * EW;
    static constexpr int CH4 = CH / 4;
    static constexpr int CV = (CH4 + 31) / 32;
    static constexpr int TOTAL = OFF_C + CH;
    static_assert(kLeadA + 3 + 7 <= 32, "alpha ring too small");
    static_assert(kLeadF + 1 + 7 <= 16, "image/F/B ring too small");
};

__device__ __forceinline__ int prow(int r) { return r + (r >> 4); }
__device__ __forceinline__ int orow8(int j) { return j + (j >> 3); }

template <bool V4>
__device__ __forceinline__ void put_block(unsigned s, const float* g, int nb) {
    if (V4) {
        cp_async16(s, g, nb);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async4(s + 4 * i, 4 * i < nb ? g + i : g, 4 * i < nb ? 4 : 0);
    }
}

// Rows streamed by one lane: alpha row (block bA), image planes and F/B planes
// (block bF).  Null pointers skip a plane.
struct RowF {
    const float* a;
    const float* i;
    const float* f;
    const float* b;
    unsigned sa, si, sf;
    int r;
};

template <int K>
__device__ __forceinline__ RowF make_rowf(const SweepJob& J, int y0, int r, bool doA, bool doI, bool doF,
                                          unsigned sbase) {
    using G = GeomF<K>;
    RowF rs;
    const int y = y0 + r;
    const bool ok = y >= 0 && y < J.h;
    const long long oi = (long long)y * J.ipitch, of = (long long)y * J.fpitch;
    rs.a = ok && doA ? J.alpha + oi : nullptr;
    rs.i = ok && doI ? J.img + oi : nullptr;
    rs.f = ok && doF ? J.fg_in + of : nullptr;
    rs.b = ok && doF ? J.bg_in + of : nullptr;
    rs.sa = sbase + 4u * unsigned(G::OFF_A + (r + 1) * 32);
    rs.si = sbase + 4u * unsigned(G::OFF_I + (r >= 0 && r < 32 ? prow(r) : 0) * 16);
    rs.sf = sbase + 4u * unsigned(G::OFF_F + (r >= 0 ? prow(r) : 0) * 16);
    rs.r = r;
    return rs;
}

template <int K, bool V4>
__device__ __forceinline__ void rowf_blocks(const RowF& rs, int bA, int bF, int w, long long is, long long fs) {
    using G = GeomF<K>;
    const int xa = 4 * bA;
    if (rs.a && xa >= 0 && xa < w) put_block<V4>(rs.sa + 4u * unsigned(xa & 31), rs.a + xa, min(4, w - xa) * 4);
    const int xf = 4 * bF;
    if (xf >= 0 && xf < w) {
        const int nb = min(4, w - xf) * 4;
        const unsigned c16 = 4u * unsigned(xf & 15);
        if (rs.i) {
#pragma unroll
            for (int c = 0; c < 3; ++c) put_block<V4>(rs.si + c16 + 4u * unsigned(c * G::IR * 16), rs.i + c * is + xf, nb);
        }
        if (rs.f) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                put_block<V4>(rs.sf + c16 + 4u * unsigned(c * G::FR * 16), rs.f + c * fs + xf, nb);
                put_block<V4>(rs.sf + c16 + 4u * unsigned((3 + c) * G::FR * 16), rs.b + c * fs + xf, nb);
            }
        }
    }
}

// Slot 0's coefficients at column x of row `lane` (alpha/image rings).
template <int K, bool G>
__device__ __forceinline__ PassC coef0(const float* sm, int lane, int x, int y, int w, int h, float eps,
                                       float omega) {
    using Gm = GeomF<K>;
    const float* ra = sm + Gm::OFF_A + (lane + 1) * 32;
    const int cn = x & 31;
    const float a = ra[cn];
    float aL = ra[(cn - 1) & 31], aR = ra[(cn + 1) & 31], aU = ra[cn - 32], aD = ra[cn + 32];
    if (G) {
        if (x <= 0) aL = a;
        if (x >= w - 1) aR = a;
        if (y <= 0) aU = a;
        if (y >= h - 1) aD = a;
    }
    const Coef3 c3 = pixel_coef3(a, aL, aR, aU, aD, eps, omega);
    PassC p;
    p.dL = c3.dL;
    p.dR = c3.dR;
    p.dU = c3.dU;
    p.dD = c3.dD;
    p.A = c3.A;
    p.A2 = c3.A2;
    p.Bn = c3.Bn;
    const float* ri = sm + Gm::OFF_I + prow(lane) * 16 + (x & 15);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float I = ri[c * Gm::IR * 16];
        p.pI[c] = __fmul_rn(c3.p, I);
        p.qI[c] = __fmul_rn(c3.q, I);
    }
    return p;
}

template <int K>
struct StateF {
    float2 outp[K][3];
    float2 rprev[K][3];
    PassC nxt;             // slot 0's coefficients for the next step
    PassC h1[K > 1 ? K - 1 : 1], h2[K > 1 ? K - 1 : 1];  // slot k's sets of the last two steps (k < K-1)
};

struct CtxF {
    const float* sm;
    float* smw;
    int lane, y0, w, h;
    bool has_up, has_down;
    int Umax;
    float* my_stream;
    float* FO;
    float* BO;
    long long ps;  // output plane stride
    int opitch;
    float eps, omega;
};

template <int K, bool G>
__device__ __forceinline__ void stepf(StateF<K>& st, const CtxF& x_, int tr) {
    using Gm = GeomF<K>;
    constexpr int OW = Gm::OW;
    const int lane = x_.lane, y0 = x_.y0, w = x_.w, h = x_.h;
    const float* sm = x_.sm;
    const bool from_up = lane == 0 && x_.has_up && (!G || (tr >= 0 && tr < x_.Umax));
    const float* cn = sm + Gm::OFF_C + (tr % kChunk) * Gm::EW;

    // F/B of lane-1 (previous step): U of slot k, R of slot k+1
    float2 recv[K][3];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            recv[k][c].x = __shfl_up_sync(kFull, st.outp[k][c].x, 1);
            recv[k][c].y = __shfl_up_sync(kFull, st.outp[k][c].y, 1);
        }
    if (from_up) {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) recv[k][c] = *reinterpret_cast<const float2*>(cn + 6 * k + 2 * c);
    }
    // coefficient sets of this step: slot 0 computed last step, slot k >= 1
    // = lane-1's slot k-1 set of two steps ago
    PassC cur[K];
    cur[0] = st.nxt;
#pragma unroll
    for (int k = 1; k < K; ++k)
#pragma unroll
        for (int i = 0; i < kPassFloats; ++i)
            pc_set(cur[k], i, __shfl_up_sync(kFull, pc_get(st.h2[k - 1], i), 1));
    if (from_up) {
#pragma unroll
        for (int k = 1; k < K; ++k)
#pragma unroll
            for (int i = 0; i < kPassFloats; ++i) pc_set(cur[k], i, cn[Gm::FBW + kPassFloats * (k - 1) + i]);
    }

    float2 nv[K][3];
    const int xs0 = tr - lane;
    const float* fr = sm + Gm::OFF_F + prow(lane) * 16;
    const float* fd = sm + Gm::OFF_F + prow(lane + 1) * 16;
    const int f0 = xs0 & 15, f1 = (xs0 + 1) & 15;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int x = xs0 - k, y = y0 + lane - k;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float2 L = st.outp[k][c], U = recv[k][c], R, D;
            if (k == 0) {
                R = make_float2(fr[c * Gm::FR * 16 + f1], fr[(3 + c) * Gm::FR * 16 + f1]);
                D = make_float2(fd[c * Gm::FR * 16 + f0], fd[(3 + c) * Gm::FR * 16 + f0]);
            } else {
                R = recv[k - 1][c];
                D = st.outp[k - 1][c];
            }
            if (G) {
                const float2 self = k == 0 ? make_float2(fr[c * Gm::FR * 16 + f0], fr[(3 + c) * Gm::FR * 16 + f0])
                                           : st.rprev[k > 0 ? k - 1 : 0][c];
                if (!(x > 0)) L = self;
                if (!(x < w - 1)) R = self;
                if (!(y > 0)) U = self;
                if (!(y < h - 1)) D = self;
            }
            nv[k][c] = apply_c(cur[k], c, L, R, U, D);
        }
    }

    // slot 0's coefficients for the next step
    st.nxt = coef0<K, G>(sm, lane, xs0 + 1, y0 + lane, w, h, x_.eps, x_.omega);

    // output ring (last sweep only)
    {
        const int x = xs0 - (K - 1);
        bool ok = true;
        if (G) ok = x >= 0 && x < w && y0 + lane - (K - 1) >= 0 && y0 + lane - (K - 1) < h;
        if (ok) {
            float* o = x_.smw + Gm::OFF_O + orow8(lane) * OW + (x & (OW - 1));
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                o[c * Gm::OR * OW] = nv[K - 1][c].x;
                o[(3 + c) * Gm::OR * OW] = nv[K - 1][c].y;
            }
        }
    }

    // boundary stream (lane 31): F/B at column u, passed sets at column u+1
    if (x_.has_down && lane == kBandRows - 1) {
        const int u = tr - 31;
        if (!G || (u >= 0 && u < x_.Umax)) {
            float* dst = x_.my_stream + size_t(u) * Gm::EW;
            float v[Gm::FBW];
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    v[6 * k + 2 * c] = nv[k][c].x;
                    v[6 * k + 2 * c + 1] = nv[k][c].y;
                }
#pragma unroll
            for (int i = 6 * K; i < Gm::FBW; ++i) v[i] = 0.0f;
#pragma unroll
            for (int i = 0; i < Gm::FBW; i += 4) st_relaxed_v4(dst + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        }
        if (K > 1 && (!G || (u >= -1 && u < x_.Umax - 1))) {
            float* dst = x_.my_stream + size_t(u + 1) * Gm::EW + Gm::FBW;
            float v[Gm::CW > 0 ? Gm::CW : 4];
#pragma unroll
            for (int k = 0; k + 1 < K; ++k)
#pragma unroll
                for (int i = 0; i < kPassFloats; ++i) v[kPassFloats * k + i] = pc_get(cur[k], i);
#pragma unroll
            for (int i = kPassFloats * (K - 1); i < Gm::CW; ++i) v[i] = 0.0f;
#pragma unroll
            for (int i = 0; i < Gm::CW; i += 4) st_relaxed_v4(dst + i, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        }
    }

    __syncwarp();
    // flush completed 8-column output row segments: four rows per step
    {
        const int col = lane & 7;
        const int jf = ((tr - (K - 1) - (OW - 1)) & (OW - 1)) + (lane & 24);
        const int xf = tr - jf - (K - 1);
        const int yf = y0 + jf - (K - 1);
        bool ok = true;
        if (G) ok = xf >= OW - 1 && xf < w && yf >= 0 && yf < h;
        if (ok) {
            const long long off = (long long)yf * x_.opitch + (xf - (OW - 1)) + col;
            const float* o = sm + Gm::OFF_O + orow8(jf) * OW + col;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                x_.FO[c * x_.ps + off] = o[c * Gm::OR * OW];
                x_.BO[c * x_.ps + off] = o[(3 + c) * Gm::OR * OW];
            }
        }
        if (G && ((w - 1) & (OW - 1)) != OW - 1) {
            const int je = tr - (K - 1) - (w - 1);
            const int x0 = (w - 1) & ~(OW - 1);
            const int ye = y0 + je - (K - 1);
            if (je >= 0 && je < 32 && ye >= 0 && ye < h && lane < w - x0) {
                const long long off = (long long)ye * x_.opitch + x0 + lane;
                const float* o = sm + Gm::OFF_O + orow8(je) * OW + lane;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    x_.FO[c * x_.ps + off] = o[c * Gm::OR * OW];
                    x_.BO[c * x_.ps + off] = o[(3 + c) * Gm::OR * OW];
                }
            }
        }
    }

#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (G) st.rprev[k][c] = recv[k][c];
            st.outp[k][c] = nv[k][c];
        }
#pragma unroll
    for (int k = 0; k + 1 < K; ++k) {
        st.h2[k] = st.h1[k];
        st.h1[k] = cur[k];
    }
}

template <int K>
__device__ __forceinline__ void chunk_load(float4 (&v)[GeomF<K>::CV], const float* up, int u0, int Umax, int lane) {
    using G = GeomF<K>;
    const int nvalid = min(kChunk, Umax - u0) * G::EW;
    const float* src = up + size_t(u0) * G::EW;
#pragma unroll
    for (int i = 0; i < G::CV; ++i) {
        const int e = lane + 32 * i;
        if (e < G::CH4 && 4 * e < nvalid) v[i] = ld_relaxed_v4(src + 4 * e);
    }
}

template <int K>
__device__ __forceinline__ void chunk_acquire(float4 (&v)[GeomF<K>::CV], const float* up, int u0, int Umax, int lane,
                                              float* chunk) {
    using G = GeomF<K>;
    const int nvalid = min(kChunk, Umax - u0) * G::EW;  // whole entries: multiples of 4
    auto complete = [&]() {
        bool ok = true;
#pragma unroll
        for (int i = 0; i < G::CV; ++i) {
            const int e = lane + 32 * i;
            if (e < G::CH4 && 4 * e < nvalid)
                ok = ok && !is_sentinel(v[i].x) && !is_sentinel(v[i].y) && !is_sentinel(v[i].z) &&
                     !is_sentinel(v[i].w);
        }
        return ok;
    };
    while (!__all_sync(kFull, complete())) {
        __nanosleep(32);
        chunk_load<K>(v, up, u0, Umax, lane);
    }
#pragma unroll
    for (int i = 0; i < G::CV; ++i) {
        const int e = lane + 32 * i;
        if (e < G::CH4 && 4 * e < nvalid) reinterpret_cast<float4*>(chunk)[e] = v[i];
    }
}

template <int K, bool V4>
__device__ __forceinline__ void run_band_f(const SweepJob& J, int q, int lane, float* sm, float eps, float omega) {
    using Gm = GeomF<K>;
    const int w = J.w, h = J.h;
    const int y0 = q * kBandRows;
    const int Umax = w + K - 1;
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    const size_t slen = sweep_full_stream_len(w, K);
    const float* up = q > 0 ? J.stream + size_t(q - 1) * slen : nullptr;
    const long long is = J.istride, fs = J.fstride;

    CtxF cx;
    cx.sm = sm;
    cx.smw = sm;
    cx.lane = lane;
    cx.y0 = y0;
    cx.w = w;
    cx.h = h;
    cx.has_up = q > 0;
    cx.has_down = q < J.nb - 1;
    cx.Umax = Umax;
    cx.my_stream = J.stream + size_t(q) * slen;
    cx.FO = J.fg_out;
    cx.BO = J.bg_out;
    cx.ps = J.ostride;
    cx.opitch = J.opitch;
    cx.eps = eps;
    cx.omega = omega;

    const RowF own = make_rowf<K>(J, y0, lane, true, true, true, sbase);
    const bool has_x = lane == 31 || lane == 0;
    const RowF ext = make_rowf<K>(J, y0, lane == 0 ? 32 : -1, has_x, false, lane == 0, sbase);

    StateF<K> st;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) st.outp[k][c] = st.rprev[k][c] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int k = 0; k + 1 < K; ++k)
#pragma unroll
        for (int i = 0; i < kPassFloats; ++i) {
            pc_set(st.h1[k], i, 0.0f);
            pc_set(st.h2[k], i, 0.0f);
        }

    {  // prologue: blocks below the first in-loop issue (t4 = -4)
        const int na = (Gm::kLeadA - own.r) >> 2, nf = (Gm::kLeadF - own.r) >> 2;
        for (int b = 0; b < max(na, nf); ++b) rowf_blocks<K, V4>(own, b < na ? b : -1, b < nf ? b : -1, w, is, fs);
        if (has_x) {
            const int ea = (Gm::kLeadA - ext.r) >> 2, ef = (Gm::kLeadF - ext.r) >> 2;
            for (int b = 0; b < max(ea, ef); ++b) rowf_blocks<K, V4>(ext, b < ea ? b : -1, b < ef ? b : -1, w, is, fs);
        }
    }
    cp_commit();
    float4 pend[Gm::CV];
    if (cx.has_up) chunk_load<K>(pend, up, 0, Umax, lane);

    const bool yband = y0 - (K - 1) <= 0 || y0 + 31 >= h - 1;
    const int fast_lo = 32 + K, fast_hi = w - 2;
    const int tend = 31 + Umax;
    for (int t4 = -4; t4 < tend; t4 += 4) {
        rowf_blocks<K, V4>(own, (t4 + 4 + Gm::kLeadA - own.r) >> 2, (t4 + 4 + Gm::kLeadF - own.r) >> 2, w, is, fs);
        if (has_x)
            rowf_blocks<K, V4>(ext, (t4 + 4 + Gm::kLeadA - ext.r) >> 2, (t4 + 4 + Gm::kLeadF - ext.r) >> 2, w, is,
                               fs);
        cp_commit();
        cp_wait<Gm::kLeadF / 4>();
        if (t4 < 0) {
            cp_wait<1>();
            __syncwarp();
            st.nxt = coef0<K, true>(sm, lane, -lane, y0 + lane, w, h, eps, omega);  // slot 0 at step 0
            continue;
        }
        if (cx.has_up && (t4 % kChunk) == 0 && t4 < Umax) {
            chunk_acquire<K>(pend, up, t4, Umax, lane, sm + Gm::OFF_C);
            if (t4 + kChunk < Umax) chunk_load<K>(pend, up, t4 + kChunk, Umax, lane);
        }
        __syncwarp();
        if (!yband && t4 >= fast_lo && t4 + 4 <= fast_hi) {
#pragma unroll
            for (int s = 0; s < 4; ++s) stepf<K, false>(st, cx, t4 + s);
        } else {
#pragma unroll 1
            for (int s = 0; s < 4; ++s) stepf<K, true>(st, cx, t4 + s);
        }
    }
    cp_wait<0>();
    __syncwarp();
}

template <int K, bool V4>
__global__ void __launch_bounds__(32) sweepf_kernel(const SweepJob* __restrict__ jobs, const int2* __restrict__ order,
                                                     int total_items, unsigned* ticket, float eps, float omega) {
    extern __shared__ float4 sm4[];
    float* sm = reinterpret_cast<float*>(sm4);
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned tk = 0;
        if (lane == 0) tk = atomicAdd(ticket, 1u);
        tk = __shfl_sync(kFull, tk, 0);
        if (tk >= unsigned(total_items)) return;
        const int2 jb = order[tk];  // (job, band)
        const SweepJob J = jobs[jb.x];
        if (V4 && !J.vec4)
            run_band_f<K, false>(J, jb.y, lane, sm, eps, omega);
        else
            run_band_f<K, V4>(J, jb.y, lane, sm, eps, omega);
    }
}

template <int K>
cudaError_t launch_f(const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket, float eps,
                     float omega, cudaStream_t s) {
    static int grid_cap = 0;
    const size_t smem = size_t(GeomF<K>::TOTAL) * sizeof(float);
    if (grid_cap == 0) {
        cudaError_t e =
            cudaFuncSetAttribute(sweepf_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweepf_kernel<K, true>, 32, smem);
        if (const char* e = std::getenv("FGM_FULL_WARPS_PER_SM")) per_sm = std::min(per_sm, std::atoi(e));  // tuning
        grid_cap = std::max(1, sms * std::max(1, per_sm));
    }
    const int grid = std::max(1, std::min(total_items, grid_cap));
    sweepf_kernel<K, true><<<grid, 32, smem, s>>>(jobs_dev, order_dev, total_items, ticket, eps, omega);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_sweep_full(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_bands,
                              unsigned* ticket, float eps, float omega, cudaStream_t s) {
    switch (K) {
        case 1: return launch_f<1>(jobs_dev, order_dev, total_bands, ticket, eps, omega, s);
        case 2: return launch_f<2>(jobs_dev, order_dev, total_bands, ticket, eps, omega, s);
        case 3: return launch_f<3>(jobs_dev, order_dev, total_bands, ticket, eps, omega, s);
        case 4: return launch_f<4>(jobs_dev, order_dev, total_bands, ticket, eps, omega, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fgm
