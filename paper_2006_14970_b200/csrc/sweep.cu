// K3: the big-level sweep kernel -- `K` fused, exact, in-place Gauss-Seidel
// scanline sweeps of one level (multilevel.cpp:81-121, repeated per
// multilevel.cpp:162-163), as a skewed-band wavefront.
//
// Dependency structure.  Pixel (x, y) of sweep k reads
// L = (x-1, y) and U = (x, y-1) of sweep k, R = (x+1, y), D = (x, y+1) and
// itself of sweep k-1.  In skewed coordinates u = x + k, v = y + k every one
// of these is (du, dv) in {(-1,0), (0,-1), (-1,-1)} -- never a positive step
// -- so:
//   * a warp owns a band of 32 skewed rows v = 32q + lane and at step t each
//     lane updates, for every k < K, pixel (t - v - k, v - k);
//   * every neighbour value comes from the lane itself or from lane-1 one
//     step earlier (registers + shfl.up), except lane 0, which reads the band
//     above's last lane from that band's boundary stream in global memory;
//   * bands depend only on the band above, and are handed out by an atomic
//     ticket in dependency order (band-major across the images of a launch),
//     so every awaited band is already resident.
//
// Boundary streams carry no flags: the buffer is filled with a NaN sentinel
// before the launch, lane 31 of band q stores its K (F_c, B_c) pairs per
// column, and band q+1 polls each 16-column chunk until no word is the
// sentinel (outputs are clamped to [0, 1], never NaN).  Each word validates
// itself, so no fences are needed on either side; the next chunk is fetched
// one chunk ahead and only re-polled if it was not complete yet.
//
// The three colour channels share only alpha (the 2x2 matrix is common to all
// channels, multilevel.hpp:37-43), so each (band, channel) is an independent
// warp: it recomputes the alpha-only coefficients (pixel_coef1) and runs the
// F_c / B_c recurrence (pixel_apply1) of its channel.
//
// Memory: each warp streams its band's rows of alpha, I_c and the initial F_c,
// B_c through per-row shared-memory rings of 32 columns, filled by cp.async
// kLead columns ahead of use; element (row r, column x) sits at ring column
// x mod 32, so the diagonal reads of a step hit 32 distinct banks and every
// ring row of a lane is a compile-time offset from its alpha row.  Outputs go
// through a 16-column ring per row and leave as coalesced 64-byte row segments
// (two rows per step) once complete.  Steps run in groups of four: loads,
// stream chunks and the border/fast decision are handled once per group.
#include <cuda_runtime.h>

#include <algorithm>

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
__device__ __forceinline__ void st_relaxed_v2(float* p, float2 v) {
    asm volatile("st.relaxed.gpu.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ bool is_sentinel(float v) { return __float_as_uint(v) == kStreamSentinel; }

// Shared-memory geometry of one (band, channel) warp, in floats.  Alpha row r
// (relative to the band) sits at OFF_A + (r + K) * 32; image row r at
// OFF_I + (r + K - 1) * 32; initial F_c / B_c row r at OFF_F / OFF_B + r * 32.
template <int K>
struct Geom {
    static constexpr int kLead = K <= 2 ? 20 : 16;  // prefetch lead in columns
    static constexpr int NA = 33 + K;               // alpha rows -K .. 32
    static constexpr int NI = 31 + K;               // image rows -(K-1) .. 31
    static constexpr int NF = 33;                   // initial F/B rows 0 .. 32
    static constexpr int OW = 16;                   // output ring columns
    static constexpr int OFF_A = 0;
    static constexpr int OFF_I = OFF_A + NA * 32;
    static constexpr int OFF_F = OFF_I + NI * 32;
    static constexpr int OFF_B = OFF_F + NF * 32;
    static constexpr int OFF_O = OFF_B + NF * 32;  // [plane F/B][lane][OW]
    static constexpr int OFF_C = OFF_O + 2 * 32 * OW;
    static constexpr int CH = kChunk * K * 2;  // one boundary-stream chunk: [u][k][F,B]
    static constexpr int CH4 = CH / 4;         // float4 per chunk (<= 32: one per lane)
    static constexpr int TOTAL = OFF_C + CH;
    static constexpr int dI = OFF_I - OFF_A - 32;      // image row r - alpha row r
    static constexpr int dF = OFF_F - OFF_A - 32 * K;  // F row r - alpha row r
    static constexpr int dB = OFF_B - OFF_A - 32 * K;  // B row r - alpha row r
    // live alpha/image window is [t-2K+2, t+2] in row-time, plus the lead
    static_assert(kLead + 2 * K + 6 <= 32, "ring too small for the prefetch lead");
    static_assert(kLead % 4 == 0, "lead must be whole 16-byte blocks");
    static_assert(CH % 4 == 0 && CH4 <= 32, "a chunk is at most one float4 per lane");
};

// The global rows a lane streams into its rings (its own row and, for some
// lanes, one extra row: alpha -K..-1, image -(K-1)..-1, F/B 32).
struct RowSrc {
    const float* a;  // alpha row (or null)
    const float* i;  // image row of channel c (or null)
    const float* f;  // initial F_c row (or null)
    const float* b;  // initial B_c row (or null)
    unsigned s;      // shared address of this row's alpha ring
    int r;           // row relative to the band
};

template <int K>
__device__ __forceinline__ RowSrc make_rowsrc(const SweepJob& J, int ch, int y0, int r, bool doA, bool doI, bool doF,
                                              unsigned sbase) {
    using G = Geom<K>;
    RowSrc rs;
    const int y = y0 + r;
    const bool ok = y >= 0 && y < J.h;
    const long long oi = (long long)y * J.ipitch, of = (long long)y * J.fpitch;
    rs.a = ok && doA ? J.alpha + oi : nullptr;
    rs.i = ok && doI ? J.img + ch * J.istride + oi : nullptr;
    rs.f = ok && doF ? J.fg_in + ch * J.fstride + of : nullptr;
    rs.b = ok && doF ? J.bg_in + ch * J.fstride + of : nullptr;
    rs.s = sbase + 4u * unsigned(G::OFF_A + (r + K) * 32);
    rs.r = r;
    return rs;
}

// cp.async of block b (columns 4b..4b+3) of one row into its rings.
template <int K, bool V4>
__device__ __forceinline__ void row_block(const RowSrc& rs, int b, int w) {
    using G = Geom<K>;
    const int x0 = 4 * b;
    if (x0 < 0 || x0 >= w) return;
    const int nb = min(4, w - x0) * 4;
    const unsigned sa = rs.s + 4u * unsigned(x0 & 31);
    auto put = [&](unsigned s, const float* row) {
        if (!row) return;
        const float* g = row + x0;
        if (V4) {
            cp_async16(s, g, nb);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) cp_async4(s + 4 * i, 4 * i < nb ? g + i : g, 4 * i < nb ? 4 : 0);
        }
    };
    put(sa, rs.a);
    put(sa + 4u * G::dI, rs.i);
    put(sa + 4u * G::dF, rs.f);
    put(sa + 4u * G::dB, rs.b);
}

// Coefficients of slot k's pixel at ring column cn (row lane-k).  G: clamp
// neighbours at the image border.
template <int K, bool G>
__device__ __forceinline__ Coef1 slot_coef(const float* sm, int aRow, int cn, int k, int x, int y, int w, int h,
                                           float eps, float omega) {
    using Gm = Geom<K>;
    const float* ra = sm + aRow - 32 * k;
    const float a = ra[cn];
    float aL = ra[(cn - 1) & 31], aR = ra[(cn + 1) & 31], aU = ra[cn - 32], aD = ra[cn + 32];
    if (G) {
        if (x <= 0) aL = a;
        if (x >= w - 1) aR = a;
        if (y <= 0) aU = a;
        if (y >= h - 1) aD = a;
    }
    return pixel_coef1(a, aL, aR, aU, aD, ra[Gm::dI + cn], eps, omega);
}

template <int K>
struct LaneState {
    float2 outp[K];   // this lane's (F_c, B_c) outputs of the previous step
    float2 rprev[K];  // what this lane received from lane-1 at the previous step (border steps)
    Coef1 co[K];      // coefficients of this step's pixels (computed one step ahead)
};

struct StepCtx {
    const float* sm;
    float* smw;
    int lane, y0, w, h;
    bool has_up, has_down;
    int Umax;
    float* my_stream;  // this band's stream (column 0)
    float* FO;
    float* BO;
    int opitch;
    float eps, omega;
};

// One wavefront step.  G: a pixel of this step or the next may be on the
// image border (clamped neighbours) or an output row segment may be partial.
template <int K, bool G>
__device__ __forceinline__ void band_step(LaneState<K>& st, const StepCtx& x_, int tr) {
    using Gm = Geom<K>;
    constexpr int OW = Gm::OW;
    const int lane = x_.lane, y0 = x_.y0, w = x_.w, h = x_.h;
    const float* sm = x_.sm;
    const int aRow = Gm::OFF_A + (lane + K) * 32;
    const int c0 = (tr - lane) & 31;

    float2 recv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        recv[k].x = __shfl_up_sync(kFull, st.outp[k].x, 1);
        recv[k].y = __shfl_up_sync(kFull, st.outp[k].y, 1);
    }
    if (lane == 0 && x_.has_up && (!G || (tr >= 0 && tr < x_.Umax))) {
        const float* cn = sm + Gm::OFF_C + (tr % kChunk) * K * 2;
#pragma unroll
        for (int k = 0; k < K; ++k) recv[k] = *reinterpret_cast<const float2*>(cn + 2 * k);
    }

    float2 nv[K];
    const int xs0 = tr - lane;  // slot-0 column
#pragma unroll
    for (int k = 0; k < K; ++k) {
        float2 L = st.outp[k], U = recv[k], R, D;
        if (k == 0) {
            const float* rf = sm + aRow;
            R = make_float2(rf[Gm::dF + ((c0 + 1) & 31)], rf[Gm::dB + ((c0 + 1) & 31)]);
            D = make_float2(rf[Gm::dF + 32 + c0], rf[Gm::dB + 32 + c0]);
        } else {
            R = recv[k - 1];
            D = st.outp[k - 1];
        }
        if (G) {
            const int x = xs0 - k, y = y0 + lane - k;
            const float2 self =
                k == 0 ? make_float2(sm[aRow + Gm::dF + c0], sm[aRow + Gm::dB + c0]) : st.rprev[k > 0 ? k - 1 : 0];
            if (!(x > 0)) L = self;
            if (!(x < w - 1)) R = self;
            if (!(y > 0)) U = self;
            if (!(y < h - 1)) D = self;
        }
        nv[k] = pixel_apply1(st.co[k], L, R, U, D);
    }

    // coefficients of the next step's pixels (alpha/image rings only)
#pragma unroll
    for (int k = 0; k < K; ++k)
        st.co[k] = slot_coef<K, G>(sm, aRow, (c0 + 1 - k) & 31, k, xs0 + 1 - k, y0 + lane - k, w, h, x_.eps,
                                   x_.omega);

    // output ring (last sweep only)
    {
        const int x = xs0 - (K - 1);
        bool ok = true;
        if (G) ok = x >= 0 && x < w && y0 + lane - (K - 1) >= 0 && y0 + lane - (K - 1) < h;
        if (ok) {
            float* o = x_.smw + Gm::OFF_O + lane * OW + (x & (OW - 1));
            o[0] = nv[K - 1].x;
            o[32 * OW] = nv[K - 1].y;
        }
    }

    // boundary stream for the band below: lane 31's K outputs of this step
    if (x_.has_down && lane == kBandRows - 1 && (!G || (tr - 31 >= 0 && tr - 31 < x_.Umax))) {
        float* dst = x_.my_stream + size_t(tr - 31) * K * 2;
        if (K % 2 == 0) {  // 16-byte aligned: u * 2K floats with K even
#pragma unroll
            for (int k = 0; k + 1 < K; k += 2)
                st_relaxed_v4(dst + 2 * k, make_float4(nv[k].x, nv[k].y, nv[k + 1].x, nv[k + 1].y));
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) st_relaxed_v2(dst + 2 * k, nv[k]);
        }
    }

    __syncwarp();
    // flush completed 16-column output row segments: rows jf (lanes 0-15) and
    // jf+16 (lanes 16-31), one coalesced 64-byte store per plane each
    {
        const int col = lane & 15;
        const int jf = ((tr - (K - 1) - (OW - 1)) & (OW - 1)) + (lane & 16);
        const int xf = tr - jf - (K - 1);  // == 15 mod 16
        const int yf = y0 + jf - (K - 1);
        bool ok = true;
        if (G) ok = xf >= OW - 1 && xf < w && yf >= 0 && yf < h;
        if (ok) {
            const long long off = (long long)yf * x_.opitch + (xf - (OW - 1)) + col;
            const float* o = sm + Gm::OFF_O + jf * OW + col;
            x_.FO[off] = o[0];
            x_.BO[off] = o[32 * OW];
        }
        if (G && ((w - 1) & (OW - 1)) != OW - 1) {  // partial last segment of a row
            const int je = tr - (K - 1) - (w - 1);
            const int x0 = (w - 1) & ~(OW - 1);
            const int ye = y0 + je - (K - 1);
            if (je >= 0 && je < 32 && ye >= 0 && ye < h && lane < w - x0) {
                const long long off = (long long)ye * x_.opitch + x0 + lane;
                const float* o = sm + Gm::OFF_O + je * OW + lane;
                x_.FO[off] = o[0];
                x_.BO[off] = o[32 * OW];
            }
        }
    }

#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (G) st.rprev[k] = recv[k];
        st.outp[k] = nv[k];
    }
}

// Poll chunk `u0 / kChunk` of the band above until every word of it is
// written; leaves it in the chunk buffer.  `v` holds a load issued earlier
// (one chunk ahead) and is re-polled only while incomplete.
template <int K>
__device__ __forceinline__ void acquire_chunk(float4 v, const float* up_stream, int u0, int Umax, int lane,
                                              float* chunk) {
    using G = Geom<K>;
    const int nvalid = min(kChunk, Umax - u0) * K * 2;  // floats
    const bool mine = lane < G::CH4 && 4 * lane < nvalid;
    auto complete = [&](float4 q) {
        if (!mine) return true;
        const int b = 4 * lane;
        return !(is_sentinel(q.x) || (b + 1 < nvalid && is_sentinel(q.y)) || (b + 2 < nvalid && is_sentinel(q.z)) ||
                 (b + 3 < nvalid && is_sentinel(q.w)));
    };
    while (!__all_sync(kFull, complete(v))) {
        __nanosleep(32);
        if (mine) v = ld_relaxed_v4(up_stream + size_t(u0) * K * 2 + 4 * lane);
    }
    if (mine) reinterpret_cast<float4*>(chunk)[lane] = v;
}

template <int K, bool V4>
__device__ __forceinline__ void run_band(const SweepJob& J, int q, int ch, int lane, float* sm, float eps,
                                         float omega) {
    using Gm = Geom<K>;
    const int w = J.w, h = J.h;
    const int y0 = q * kBandRows;
    const int Umax = w + K - 1;
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    const size_t slen = sweep_stream_len(w, K);
    const int sid = q * 3 + ch;  // stream index of this (band, channel)
    const float* up_stream = q > 0 ? J.stream + size_t(sid - 3) * slen : nullptr;

    StepCtx cx;
    cx.sm = sm;
    cx.smw = sm;
    cx.lane = lane;
    cx.y0 = y0;
    cx.w = w;
    cx.h = h;
    cx.has_up = q > 0;
    cx.has_down = q < J.nb - 1;
    cx.Umax = Umax;
    cx.my_stream = J.stream + size_t(sid) * slen;
    cx.FO = J.fg_out + (long long)ch * J.ostride;
    cx.BO = J.bg_out + (long long)ch * J.ostride;
    cx.opitch = J.opitch;
    cx.eps = eps;
    cx.omega = omega;

    // rows this lane streams
    const RowSrc own = make_rowsrc<K>(J, ch, y0, lane, true, true, true, sbase);
    const bool has_x = lane >= 32 - K || lane == 0;
    const RowSrc ext = make_rowsrc<K>(J, ch, y0, lane == 0 ? 32 : lane - 32, has_x, lane >= 33 - K, lane == 0, sbase);

    LaneState<K> st;
#pragma unroll
    for (int k = 0; k < K; ++k) st.outp[k] = st.rprev[k] = make_float2(0.0f, 0.0f);

    // prologue: blocks below the first in-loop issue (t4 = -4 loads block
    // (kLead - r) / 4 of row r)
    for (int b = 0; b < ((Gm::kLead - own.r) >> 2); ++b) row_block<K, V4>(own, b, w);
    if (has_x)
        for (int b = 0; b < ((Gm::kLead - ext.r) >> 2); ++b) row_block<K, V4>(ext, b, w);
    cp_commit();
    // the band above's first chunk, polled when needed
    float4 pend = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool lane_ch = lane < Gm::CH4;
    if (cx.has_up && lane_ch) pend = ld_relaxed_v4(up_stream + 4 * lane);

    // Border groups: bands touching row 0 or h-1, else the first and last ~32
    // steps.  Fast groups need no neighbour clamping and no bounds checks.
    const bool yband = y0 - (K - 1) <= 0 || y0 + 31 >= h - 1;
    const int fast_lo = 32 + K, fast_hi = w - 2;  // a step tr is fast iff fast_lo <= tr < fast_hi
    const int tend = 31 + Umax;                   // lane 31's last column is Umax-1
    for (int t4 = -4; t4 < tend; t4 += 4) {
        row_block<K, V4>(own, (t4 + 4 + Gm::kLead - own.r) >> 2, w);
        if (has_x) row_block<K, V4>(ext, (t4 + 4 + Gm::kLead - ext.r) >> 2, w);
        cp_commit();
        cp_wait<Gm::kLead / 4 - 1>();
        if (t4 < 0) {
            cp_wait<1>();  // the prologue group
            __syncwarp();
            const int aRow = Gm::OFF_A + (lane + K) * 32;
#pragma unroll
            for (int k = 0; k < K; ++k)  // coefficients of step 0
                st.co[k] = slot_coef<K, true>(sm, aRow, (-lane + 1 - k - 1) & 31, k, -lane - k, y0 + lane - k, w, h,
                                              eps, omega);
            continue;
        }
        if (cx.has_up && (t4 % kChunk) == 0 && t4 < Umax) {
            acquire_chunk<K>(pend, up_stream, t4, Umax, lane, sm + Gm::OFF_C);
            if (t4 + kChunk < Umax && lane_ch)  // prefetch the next chunk
                pend = ld_relaxed_v4(up_stream + size_t(t4 + kChunk) * K * 2 + 4 * lane);
        }
        __syncwarp();
        if (!yband && t4 >= fast_lo && t4 + 4 <= fast_hi) {
#pragma unroll
            for (int s = 0; s < 4; ++s) band_step<K, false>(st, cx, t4 + s);
        } else {
#pragma unroll 1
            for (int s = 0; s < 4; ++s) band_step<K, true>(st, cx, t4 + s);
        }
    }
    cp_wait<0>();
    __syncwarp();
}

template <int K, bool V4>
__global__ void __launch_bounds__(32) sweep_kernel(const SweepJob* __restrict__ jobs, const int2* __restrict__ order,
                                                    int total_items, unsigned* ticket, float eps, float omega) {
    extern __shared__ float4 sm4[];
    float* sm = reinterpret_cast<float*>(sm4);
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned tk = 0;
        if (lane == 0) tk = atomicAdd(ticket, 1u);
        tk = __shfl_sync(kFull, tk, 0);
        if (tk >= unsigned(total_items)) return;
        const int2 jb = order[tk];  // (job, band * 3 + channel)
        const SweepJob J = jobs[jb.x];
        if (V4 && !J.vec4) {
            run_band<K, false>(J, jb.y / 3, jb.y % 3, lane, sm, eps, omega);
        } else {
            run_band<K, V4>(J, jb.y / 3, jb.y % 3, lane, sm, eps, omega);
        }
    }
}

template <int K>
cudaError_t launch_sweep_k(const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket,
                           float eps, float omega, cudaStream_t s) {
    static int grid_cap = 0;
    const size_t smem = size_t(Geom<K>::TOTAL) * sizeof(float);
    if (grid_cap == 0) {
        cudaError_t e =
            cudaFuncSetAttribute(sweep_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<K, true>, 32, smem);
        grid_cap = std::max(1, sms * std::max(1, per_sm));
    }
    const int grid = std::max(1, std::min(total_items, grid_cap));
    sweep_kernel<K, true><<<grid, 32, smem, s>>>(jobs_dev, order_dev, total_items, ticket, eps, omega);
    return cudaGetLastError();
}

__global__ void stream_fill_kernel(const SweepJob* __restrict__ jobs, int K, bool full) {
    const SweepJob J = jobs[blockIdx.y];
    const size_t n = size_t(J.nb) * (full ? sweep_full_stream_len(J.w, K) : 3 * sweep_stream_len(J.w, K)) / 4;
    float4* p = reinterpret_cast<float4*>(J.stream);
    const float s = __uint_as_float(kStreamSentinel);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = make_float4(s, s, s, s);
}

}  // namespace

cudaError_t launch_stream_fill(const SweepJob* jobs_dev, int njobs, int K, bool full, size_t max_floats,
                               cudaStream_t s) {
    if (njobs <= 0) return cudaSuccess;
    const int gx = int(std::min<size_t>(std::max<size_t>((max_floats / 4 + 255) / 256, 1), 64));
    stream_fill_kernel<<<dim3(gx, njobs), 256, 0, s>>>(jobs_dev, K, full);
    return cudaGetLastError();
}

int sweep_supported_k(int K) { return K >= 1 && K <= 4; }

size_t sweep_smem_bytes(int K) {
    switch (K) {
        case 1: return Geom<1>::TOTAL * sizeof(float);
        case 2: return Geom<2>::TOTAL * sizeof(float);
        case 3: return Geom<3>::TOTAL * sizeof(float);
        case 4: return Geom<4>::TOTAL * sizeof(float);
        default: return 0;
    }
}

cudaError_t launch_sweep(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket,
                         float eps, float omega, cudaStream_t s) {
    switch (K) {
        case 1: return launch_sweep_k<1>(jobs_dev, order_dev, total_items, ticket, eps, omega, s);
        case 2: return launch_sweep_k<2>(jobs_dev, order_dev, total_items, ticket, eps, omega, s);
        case 3: return launch_sweep_k<3>(jobs_dev, order_dev, total_items, ticket, eps, omega, s);
        case 4: return launch_sweep_k<4>(jobs_dev, order_dev, total_items, ticket, eps, omega, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fgm
