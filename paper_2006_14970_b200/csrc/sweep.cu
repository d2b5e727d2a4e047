// K3: the big-level sweep kernel -- `K` fused, exact, in-place Gauss-Seidel
// scanline sweeps of one level (multilevel.cpp:81-121, repeated per
// multilevel.cpp:162-163), as a skewed-band wavefront.
//
// Dependency structure.  Pixel (x, y) of sweep k reads
// L = (x-1, y) and U = (x, y-1) of sweep k, R = (x+1, y), D = (x, y+1) and
// itself of sweep k-1.  In skewed coordinates u = x + k, v = y + k every one
// of these is (du, dv) in {(-1,0), (0,-1), (-1,-1)} -- never a positive step.
//
// Geometry (round 2).  A warp owns a band of 64 skewed rows; lane j owns the
// two consecutive rows r = 2j, 2j+1 (band-relative) and at step t updates, for
// every slot k < K, pixel (t - r - k, y0 + r - k) of each row.  Every value a
// step needs was produced at the previous step: by the same row (L, and D of
// slot k >= 1), by the row above (U, and R of slot k >= 1) -- for row 2j+1
// that is row 2j of the same lane, for row 2j the previous lane's row 2j-1
// (shfl.up), for lane 0 the band above's last row, read from that band's
// boundary stream.  The 2 x K pixel updates of a step are independent.
//
// Coefficients.  The 2x2 matrix depends on alpha only and is common to the
// three channels and to the K sweeps (multilevel.hpp:37-43): slot k of row
// 2j+1 updates the pixel slot k-1 of row 2j updated two steps earlier (pixel
// (x, y) of sweep k runs at step x + y + 2k), so its coefficients are that
// step's, delayed in registers; only row 2j's slots k >= 1 recompute theirs.  Edge weights are reused along the rows (dL = the
// previous step's dR) and down the lane (row 2j+1's dU = row 2j's previous dD).
//
// Memory staging.  Each warp streams its band's rows of alpha, I_c and the
// initial F_c, B_c through per-row shared-memory rings of 32 columns, refilled
// in 16-column (64-byte) row segments: four lanes per row segment, eight row
// segments per cp.async instruction (per-lane 16-byte segments of 32
// different rows cap at 2.7 TB/s on B200, 64-byte segments reach 5.8-6.3 TB/s
// at this kernel's occupancy; profiles/r02/membench*.txt).  A row's next
// segment is issued as soon as the segment it replaces is no longer read; the
// row offsets of the two lanes' rows make the refills of a 4-step group fall
// on 4 consecutive rows of every 16-row block.  Outputs go through a 16-column
// ring per row and leave as 64-byte row segments (two rows per store).
//
// Boundary streams carry no flags: the buffer is filled with a NaN sentinel
// before the launch, lane 31 stores its last row's K (F_c, B_c) pairs per
// column, and the band below polls each chunk of columns until no word is the
// sentinel (outputs are clamped to [0, 1], never NaN).  Each word validates
// itself, so no fences are needed on either side; the waits are bounded
// (timeout -> error, not a hang).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "fgm_device.cuh"
#include "fgm_internal.h"

namespace fgm {
namespace {

constexpr int R = 2;           // rows per lane
constexpr int BR = kBandRows;  // band rows
static_assert(BR == 32 * R, "a band is 32 lanes x R rows");

__device__ __forceinline__ void cp_async16(unsigned sdst, const float* gsrc, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gsrc), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16f(unsigned sdst, const float* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
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
// Boundary-stream stores need no ordering against this warp's other memory
// operations (every word validates itself), hence no "memory" clobber.
__device__ __forceinline__ void st_relaxed_v4(float* p, float4 v) {
    asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
}
__device__ __forceinline__ void st_relaxed_v2(float* p, float2 v) {
    asm volatile("st.relaxed.gpu.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y));
}
extern __shared__ float4 sweep_sm4[];
__device__ __forceinline__ void sts4(int i, float4 v) { reinterpret_cast<float4*>(reinterpret_cast<float*>(sweep_sm4) + i)[0] = v; }
__device__ __forceinline__ void stg(float* p, float v) { __stcg(p, v); }
__device__ __forceinline__ bool is_sentinel(float v) { return __float_as_uint(v) == kStreamSentinel; }

// Shared-memory geometry of one (band, channel) warp, in floats.
//   rings: [plane][ring row][32 columns], column x at x & 31; ring row = band
//          row - L_p (alpha rows -K..64, image rows -(K-1)..63, F/B rows
//          0..64), refilled in 16-column (64-byte) segments.  (16-column F/B
//          rings with 8-column segments -- F and B are read at one column per
//          row and step -- would fit 6 warps per SM, but leave one 4-step
//          group of lead: measured 20% slower, the refill wait stalls on DRAM
//          latency even with L2 prefetches; profiles/r02/k3_v2_notes.txt)
//   output ring: [F/B][orow(r)][16 columns]; chunk buffer: [column][k][F, B]
// Read window of ring row r at step t, relative to t - r: alpha [MA, 1],
// image [MI, 0], F/B [1, 1] (MA, MI: the recomputed slots and the rows below
// reading their upper neighbour).  A segment is refilled when the segment
// whose ring slot it takes leaves the window.
template <int K, int CK>
struct Geom {
    static constexpr int RW = 32, RWF = 32;
    static constexpr int LA = -K, NA = BR + 1 + K;
    static constexpr int LI = -(K - 1), NI = BR + K - 1;
    static constexpr int NF = BR + 1;  // F/B rows 0 .. 64
    static constexpr int OFF_A = 0;
    static constexpr int OFF_I = OFF_A + NA * RW;
    static constexpr int OFF_F = OFF_I + NI * RW;
    static constexpr int OFF_B = OFF_F + NF * RWF;
    static constexpr int OW = 16;
    static constexpr int OPL = (BR + BR / 16) * OW;
    static constexpr int OFF_O = OFF_B + NF * RWF;
    static constexpr int OFF_C = OFF_O + 2 * OPL;
    static constexpr int CH = CK * K * 2;  // one boundary-stream chunk: [column][k][F, B]
    static constexpr int CH4 = CH / 4;     // float4 per chunk (<= 32: one per lane)
    static constexpr int TOTAL = OFF_C + CH;
    // per plane p (0 alpha, 1 image, 2 F, 3 B): segment width, window
    static constexpr int sw(int p) { return 16; }
    static constexpr int mlo(int p) { return p == 0 ? (K >= 2 ? -(2 * K - 1) : -1) : p == 1 ? -2 * (K - 1) : 1; }
    static constexpr int mhi(int p) { return p == 1 ? 0 : 1; }
    // the refill phase: issue time - free time, making the rows of a 4-step
    // group's refills 4 consecutive rows of each segment-width block
    static constexpr int phase(int p) { return ((mlo(p) % 4) + 4) % 4; }
    // steps from a refill's issue to its first read
    static constexpr int lead(int p) { return sw(p) - mhi(p) + mlo(p) - phase(p); }
    static constexpr int minlead() {
        return lead(0) < lead(1) ? (lead(0) < lead(2) ? lead(0) : lead(2)) : (lead(1) < lead(2) ? lead(1) : lead(2));
    }
    // a group waits for the refills issued two groups back when every lead is
    // >= 8 steps, else for those of the previous group (then >= 4 steps)
    static constexpr int WAITN = minlead() >= 8 ? 1 : 0;
    static_assert(CH % 4 == 0 && CH4 <= 32, "a chunk is at most one float4 per lane");
    static_assert(minlead() >= 4, "read window too wide for the ring");
};

__device__ __forceinline__ constexpr int orow(int r) { return r + (r >> 4); }

// The rank-one coefficients (fgm_device.cuh, pixel_coefr_dl) from the four
// edge weights: the same operations in the same order.
__device__ __forceinline__ CoefR coef_w(float a, float dL, float dR, float dU, float dD, float I) {
    CoefR co;
    co.dL = dL;
    co.dR = dR;
    co.dU = dU;
    co.dD = dD;
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(dL, dR), dU), dD);
    co.u = pk2(a, __fsub_rn(1.0f, a));
    const float2 uu = upk2(mul2(co.u, co.u));
    const float Dn = __fadd_rn(__fadd_rn(uu.x, uu.y), S);
    co.iS = rcp_approx(S);
    const float iD = rcp_approx(Dn);
    co.pq = mul2(pk2(iD, iD), co.u);
    co.I = I;
    return co;
}

template <int K>
struct LaneState {
    float2 o[R][K];  // (F_c, B_c) of the previous step, per row and slot
    float2 o2[K];    // row 2j's outputs two steps back (border self values of row 2j+1)
    float2 rvp[K];   // the previous step's values from the row above row 2j
    CoefR cp1[K];    // row 2j's coefficients of the previous step
    CoefR cp2[K];    // and of the step before (row 2j+1's slots 1..K-1)
    float aRp[R];    // the previous step's right-neighbour alpha per row (this step's alpha)
    float dRp[R];    // the previous step's slot-0 dR per row (this step's dL)
    float dDp;       // row 2j's previous slot-0 dD (row 2j+1's dU)
    float dRr[K];    // row 2j's recomputed slots: the previous dR
    float aU0p, a0p; // K = 2: the previous step's alpha above row 2j and row 2j's alpha
    float2 FRp[R];   // the previous step's initial (F, B) right neighbours: this step's slot-0 own values
};

struct StepCtx {
    int lane, y0, w, h, Umax;
    unsigned lb4;      // byte offset of ring row 2j in a plane (256 * lane: bits >= 8)
    unsigned ob4;      // byte offset of output-ring row orow(2j) (bits >= 7)
    unsigned flb4;     // flush: byte offset of output-ring row 17 * (lane >> 4), column lane & 15
    bool has_up, has_down;
    float* my_stream;  // this band's stream (column 0)
    float* gF;         // flush base, F plane: FO + 16 (lane >> 4) (opitch - 1) + (lane & 15) - K - 14
    float* gB;
    int op1;           // opitch - 1
    unsigned ytop, ybot;  // YE: bit (i * K + k): pixel row y <= 0 / y >= h - 1 (constant over the band)
    float eps, omega;
};

__device__ __forceinline__ float2 ldsb2(unsigned off) {
    return *reinterpret_cast<const float2*>(reinterpret_cast<const char*>(sweep_sm4) + off);
}
__device__ __forceinline__ void stsb2(unsigned off, float2 v) {
    *reinterpret_cast<float2*>(reinterpret_cast<char*>(sweep_sm4) + off) = v;
}
// (F, B) from the previous lane as one 64-bit shuffle: lands in a register pair
__device__ __forceinline__ float2 shfl_up_pair(float2 v) {
    return upk2(__shfl_up_sync(kFull, pk2(v), 1));
}
__device__ __forceinline__ float ldsb(unsigned off) {
    return *reinterpret_cast<const float*>(reinterpret_cast<const char*>(sweep_sm4) + off);
}

// Step variants: X = 0 interior columns, 1 left border region (some x <= 0),
// 2 right border region (some x >= w - 1), 3 both; YE: a band touching the
// top or bottom row.  Without X and YE every pixel, flushed segment and stream
// slot is inside the image: no clamps, no bounds checks.
template <int K, int CK, int X, bool YE>
__device__ __forceinline__ void band_step(LaneState<K>& st, const StepCtx& x_, int c4g, int t4, int s) {
    using G = Geom<K, CK>;
    constexpr bool XLm = X & 1, XRm = X & 2, XE = X != 0, BD = XE || YE;
    const int lane = x_.lane;
    const int t = t4 + s;
    const float eps = x_.eps, omega = x_.omega;
    // byte offset of ring row 2j, column (t - 2j + e)
    auto C = [&](int e) { return x_.lb4 | (unsigned(c4g + 4 * (s + e)) & 124u); };
    auto A = [&](int d) { return unsigned(4 * (G::OFF_A + (d - G::LA) * G::RW)); };
    auto Ip = [&](int d) { return unsigned(4 * (G::OFF_I + (d - G::LI) * G::RW)); };
    auto CF = C;
    auto Fp = [&](int d) { return unsigned(4 * (G::OFF_F + d * G::RWF)); };
    auto Bp = [&](int d) { return unsigned(4 * (G::OFF_B + d * G::RWF)); };

    // values from the row above row 2j: shfl.up of row 2j+1, lane 0 from the chunk
    float2 rv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) rv[k] = shfl_up_pair(st.o[1][k]);
    if (lane == 0 && x_.has_up) {
        const unsigned cn = unsigned(4 * G::OFF_C + (t & (CK - 1)) * K * 8);
#pragma unroll
        for (int k = 0; k < K; ++k) rv[k] = ldsb2(cn + 8 * k);
    }

    // slot-0 loads: row 2j (x0 = t - 2j), row 2j+1 (x1 = x0 - 1)
    const float aR0 = ldsb(C(1) + A(0)), aR1 = ldsb(C(0) + A(1));
    const float I0 = ldsb(C(0) + Ip(0)), I1 = ldsb(C(-1) + Ip(1));
    const float2 FR0 = make_float2(ldsb(CF(1) + Fp(0)), ldsb(CF(1) + Bp(0)));
    const float2 FR1 = make_float2(ldsb(CF(0) + Fp(1)), ldsb(CF(0) + Bp(1)));
    const float aU0 = ldsb(C(0) + A(-1));
    const float aD1 = ldsb(C(-1) + A(2));
    const float2 FD1 = make_float2(ldsb(CF(-1) + Fp(2)), ldsb(CF(-1) + Bp(2)));

    const int x0 = t - 2 * lane;
    const int w = x_.w;
    auto top = [&](int i, int k) { return YE && ((x_.ytop >> (i * K + k)) & 1u); };
    auto bot = [&](int i, int k) { return YE && ((x_.ybot >> (i * K + k)) & 1u); };
    auto xlo = [&](int x) { return XLm && x <= 0; };
    auto xhi = [&](int x) { return XRm && x >= w - 1; };

    // slot-0 coefficients
    const float a0 = st.aRp[0], a1 = st.aRp[1];
    float dL0 = st.dRp[0], dL1 = st.dRp[1], dU1 = st.dDp;
    float aR0c = aR0, aR1c = aR1, aU0c = aU0, aD0c = aR1, aD1c = aD1;
    if (xlo(x0)) dL0 = eps;
    if (xlo(x0 - 1)) dL1 = eps;
    if (xhi(x0)) aR0c = a0;
    if (xhi(x0 - 1)) aR1c = a1;
    if (top(0, 0)) aU0c = a0;
    if (bot(0, 0)) aD0c = a0;
    if (top(1, 0)) dU1 = eps;
    if (bot(1, 0)) aD1c = a1;
    const float dR0 = edge_weight(a0, aR0c, eps, omega), dU0 = edge_weight(a0, aU0c, eps, omega);
    const float dD0 = edge_weight(a0, aD0c, eps, omega), dR1 = edge_weight(a1, aR1c, eps, omega);
    const float dD1 = edge_weight(a1, aD1c, eps, omega);
    CoefR co[R][K];
    co[0][0] = coef_w(a0, dL0, dR0, dU0, dD0, I0);
    co[1][0] = coef_w(a1, dL1, dR1, dU1, dD1, I1);

    // row 2j's slots k >= 1: pixel (x0 - k, band row 2j - k), recomputed (K = 2:
    // three of its four alphas are this and the previous step's)
    float dRr[K];
#pragma unroll
    for (int k = 1; k < K; ++k) {
        float a, aR, aD;
        if (K == 2) {
            a = st.aU0p;
            aR = aU0;
            aD = st.a0p;
        } else {
            a = ldsb(C(-k) + A(-k));
            aR = ldsb(C(-k + 1) + A(-k));
            aD = ldsb(C(-k) + A(-k + 1));
        }
        float aU = ldsb(C(-k) + A(-k - 1));
        const float I = ldsb(C(-k) + Ip(-k));
        float dL = st.dRr[k];
        if (xlo(x0 - k)) dL = eps;
        if (xhi(x0 - k)) aR = a;
        if (top(0, k)) aU = a;
        if (bot(0, k)) aD = a;
        const float dR = edge_weight(a, aR, eps, omega);
        co[0][k] = coef_w(a, dL, dR, edge_weight(a, aU, eps, omega), edge_weight(a, aD, eps, omega), I);
        dRr[k] = dR;
        co[1][k] = st.cp2[k - 1];
    }

    // the updates
    float2 nv[R][K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        {  // row 2j
            float2 L = st.o[0][k], U = rv[k];
            float2 Rn = k ? rv[k > 0 ? k - 1 : 0] : FR0;
            float2 D = k ? st.o[0][k > 0 ? k - 1 : 0] : FR1;
            if (BD) {
                const float2 self = k ? st.rvp[k > 0 ? k - 1 : 0] : st.FRp[0];
                if (xlo(x0 - k)) L = self;
                if (xhi(x0 - k)) Rn = self;
                if (top(0, k)) U = self;
                if (bot(0, k)) D = self;
            }
            nv[0][k] = pixel_applyr(co[0][k], L, Rn, U, D);
        }
        {  // row 2j+1
            float2 L = st.o[1][k], U = st.o[0][k];
            float2 Rn = k ? st.o[0][k > 0 ? k - 1 : 0] : FR1;
            float2 D = k ? st.o[1][k > 0 ? k - 1 : 0] : FD1;
            if (BD) {
                const float2 self = k ? st.o2[k > 0 ? k - 1 : 0] : st.FRp[1];
                if (xlo(x0 - 1 - k)) L = self;
                if (xhi(x0 - 1 - k)) Rn = self;
                if (top(1, k)) U = self;
                if (bot(1, k)) D = self;
            }
            nv[1][k] = pixel_applyr(co[1][k], L, Rn, U, D);
        }
    }

    // output ring (last sweep only), row orow(2j + i), column x & 15, (F, B)
    // interleaved.  Pixels outside the image land in slots that are
    // rewritten or never flushed.
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const unsigned o = (x_.ob4 + 128u * i) | (unsigned(2 * (c4g + 4 * (s - i - (K - 1)))) & 120u);
        stsb2(o, nv[i][K - 1]);
    }

    // boundary stream for the band below: the last row's K outputs
    if (x_.has_down && lane == 31) {
        const int u = t - (BR - 1);
        if ((!XLm || u >= 0) && (!XRm || u < x_.Umax)) {
            float* dst = x_.my_stream + size_t(u) * K * 2;
            if (K % 2 == 0) {
#pragma unroll
                for (int k = 0; k + 1 < K; k += 2)
                    st_relaxed_v4(dst + 2 * k, make_float4(nv[1][k].x, nv[1][k].y, nv[1][k + 1].x, nv[1][k + 1].y));
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) st_relaxed_v2(dst + 2 * k, nv[1][k]);
            }
        }
    }

    __syncwarp();
    // flush the 16-column output row segments completed by this step: rows
    // r = rho + 16 beta (beta = 0..3), lanes 0-15 / 16-31 two rows per store;
    // column x = t - K - 14 - r + (lane & 15)
    {
        const int rho = (t - K - 14) & 15;
        const unsigned lo = x_.flb4 + 128u * unsigned(rho);
        const int off0 = rho * x_.op1 + t;
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
            bool ok = true;
            if (XE || YE) {
                const int r = rho + 16 * (2 * hb + (lane >> 4));
                const int x = t - K - 14 - r + (lane & 15);
                if (XLm) ok = ok && x - (lane & 15) >= 0;
                if (XRm) ok = ok && x < w;
                if (YE) ok = ok && unsigned(x_.y0 + r - (K - 1)) < unsigned(x_.h);
            }
            if (ok) {  // (off >= 0 whenever ok: one IMAD.WIDE.U32 per address)
                const unsigned off = unsigned(off0 + hb * 32 * x_.op1);
                const float2 v = ldsb2(lo + hb * 34u * 128u);
                stg(x_.gF + off, v.x);
                stg(x_.gB + off, v.y);
            }
        }
        if (XRm && ((w - 1) & (G::OW - 1)) != G::OW - 1) {  // the partial last segment of a row
            const int re = t - (K - 1) - (w - 1);
            const int xb = (w - 1) & ~(G::OW - 1);
            const int y = x_.y0 + re - (K - 1);
            if (re >= 0 && re < BR && y >= 0 && y < x_.h && lane < w - xb) {
                // (lanes < 16: gF = FO + lane - K - 14)
                const int off = re * (x_.op1 + 1) + xb + K + 14;
                const float2 v = ldsb2(unsigned(4 * G::OFF_O + 8 * (orow(re) * G::OW + lane)));
                stg(x_.gF + off, v.x);
                stg(x_.gB + off, v.y);
            }
        }
    }

    // every lane's flush reads are done before the next step's output-ring
    // stores reuse the slots (lanes of a diverged warp may run ahead)
    __syncwarp();
    // carry
#pragma unroll
    for (int k = 0; k < K; ++k) {
        st.o2[k] = st.o[0][k];
        st.rvp[k] = rv[k];
        st.o[0][k] = nv[0][k];
        st.o[1][k] = nv[1][k];
        st.cp2[k] = st.cp1[k];
        st.cp1[k] = co[0][k];
        if (k >= 1) st.dRr[k] = dRr[k];
    }
    st.aU0p = aU0;
    st.a0p = a0;
    st.FRp[0] = FR0;
    st.FRp[1] = FR1;
    st.aRp[0] = aR0;
    st.aRp[1] = aR1;
    st.dRp[0] = dR0;
    st.dRp[1] = dR1;
    st.dDp = dD0;
}

// ---- ring refills -----------------------------------------------------------
// Plane p (0 alpha, 1 image, 2 F, 3 B; segment width SW, ring width 2 SW) of
// band row r: segment n (columns SW n .. SW n + SW - 1) is issued at step
// SW (n-1) + r - mlo + phase, when the segment n-2 in its ring slot has left
// the read window.  In the group of steps [t4, t4+4) that is, with
// Z = t4 + mlo - phase (a multiple of 4): rows r = SW beta + (Z mod SW) + rho
// (rho = 0..3) get segment n = (Z div SW) + 1 - beta.  A cp.async instruction
// covers 32 / SW * 4 ... row segments: lanes = (block, rho, 16-byte piece).
struct RefillSrc {
    const float* base[4];  // plane row 0 (image row y0), column 0
    int pitch[4];
};

template <int K, int CK>
__device__ __forceinline__ constexpr int plane_lo(int p) {
    using G = Geom<K, CK>;
    return p == 0 ? G::LA : p == 1 ? G::LI : 0;
}
__device__ __forceinline__ constexpr int plane_hi(int p) { return p == 1 ? BR - 1 : BR; }
template <int K, int CK>
__device__ __forceinline__ constexpr int plane_off(int p) {
    using G = Geom<K, CK>;
    return p == 0 ? G::OFF_A : p == 1 ? G::OFF_I : p == 2 ? G::OFF_F : G::OFF_B;
}
template <int K, int CK>
__device__ __forceinline__ constexpr int plane_rows(int p) {
    using G = Geom<K, CK>;
    return p == 0 ? G::NA : p == 1 ? G::NI : G::NF;
}
__device__ __forceinline__ constexpr int plane_rw(int p) { return 32; }

// One 16-byte piece (4 columns from c) of plane P, band row r, with every check.
template <int K, bool V4, int CK, int P>
__device__ __forceinline__ void put_piece(const RefillSrc& S, unsigned sbase, int r, int c, int y0, int w, int h) {
    constexpr int RWp = plane_rw(P);
    if (r < plane_lo<K, CK>(P) || r > plane_hi(P) || c < 0 || c >= w) return;
    const int y = y0 + r;
    if (y < 0 || y >= h) return;
    const float* g = S.base[P] + (long long)r * S.pitch[P] + c;
    const unsigned d = sbase + 4u * unsigned(plane_off<K, CK>(P) + (r - plane_lo<K, CK>(P)) * RWp + (c & (RWp - 1)));
    const int nb = min(w - c, 4);
    if (V4) {
        cp_async16(d, g, nb * 4);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async4(d + 4 * i, i < nb ? g + i : g, i < nb ? 4 : 0);
    }
}

// Lane roles of a refill instruction of plane P: piece q of the segment,
// row rho of the 4-row group, block bsub of the instruction's blocks.
template <int P>
struct RefillLane {
    static constexpr int SW = 16, PPS = SW / 4, BPI = 8 / PPS;  // blocks per instruction
    int q, rho, bsub;
    __device__ __forceinline__ explicit RefillLane(int lane) : q(lane % PPS), rho((lane / PPS) & 3), bsub(lane / (4 * PPS)) {}
};

// The refills of plane P in group t4, every piece checked (band edges, image
// edges, jobs without 16-byte aligned rows).
template <int K, bool V4, int CK, int P>
__device__ __forceinline__ void refill_checked_p(const RefillSrc& S, unsigned sbase, int t4, int lane, int y0, int w,
                                                 int h) {
    using G = Geom<K, CK>;
    using RL = RefillLane<P>;
    constexpr int SW = RL::SW;
    const RL L(lane);
    const int Z = t4 + G::mlo(P) - G::phase(P);
    const int zr = Z & (SW - 1), zh = Z >> (SW == 16 ? 4 : 3);
    // beta = -1 .. 64 / SW covers band rows -SW .. 64 + SW - 1
#pragma unroll
    for (int b0 = -RL::BPI; b0 <= BR / SW; b0 += RL::BPI) {
        const int beta = b0 + L.bsub;
        const int r = SW * beta + zr + L.rho;
        const int c0 = SW * (zh + 1 - beta);
        if (c0 >= 2 * SW) put_piece<K, V4, CK, P>(S, sbase, r, c0 + 4 * L.q, y0, w, h);
    }
}
template <int K, bool V4, int CK>
__device__ __forceinline__ void refill_checked(const RefillSrc& S, unsigned sbase, int t4, int lane, int y0, int w,
                                               int h) {
    refill_checked_p<K, V4, CK, 0>(S, sbase, t4, lane, y0, w, h);
    refill_checked_p<K, V4, CK, 1>(S, sbase, t4, lane, y0, w, h);
    refill_checked_p<K, V4, CK, 2>(S, sbase, t4, lane, y0, w, h);
    refill_checked_p<K, V4, CK, 3>(S, sbase, t4, lane, y0, w, h);
}

__device__ __forceinline__ void cp_async16_if(unsigned sdst, const float* gsrc, bool pred) {
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16;\n}" ::"r"(sdst),
                 "l"(gsrc), "r"(unsigned(pred))
                 : "memory");
}

// The main row blocks of plane P in group t4 (band rows 0..63, two
// instructions 32 rows apart), for jobs with 16-byte aligned rows.  CHECK:
// pieces outside the image (rows of a band at the top or bottom, columns at
// the row ends) or before segment 2 (the prologue's) are predicated off;
// without CHECK every piece is inside.
template <int K, int CK, int P, bool CHECK>
__device__ __forceinline__ void refill_main_p(const RefillSrc& S, int lo_off, unsigned ss, int t4, int lane, int y0,
                                              int w, int h) {
    using G = Geom<K, CK>;
    using RL = RefillLane<P>;
    constexpr int SW = RL::SW, RWp = 2 * SW;
    const RL L(lane);
    const int Z = t4 + G::mlo(P) - G::phase(P);
    const int zr = Z & (SW - 1), zh = Z >> 4;
    // 32-bit element offsets from the band's plane base (rows 0 .. 63, >= 0
    // whenever the piece is copied): one IMAD.WIDE.U32 per address
    const unsigned off = unsigned(lo_off + zr * S.pitch[P] + SW * zh);
    const float* g = S.base[P] + off;
    const float* g2 = S.base[P] + (off + unsigned(32 * S.pitch[P] - 32));
    const unsigned d = ss + 4u * unsigned(plane_off<K, CK>(P) - plane_lo<K, CK>(P) * RWp) +
                       unsigned(zr * RWp * 4 + 4 * SW * ((zh + 1 + L.bsub) & 1));
    const unsigned d2 = d + 4u * 32u * RWp;
    if (CHECK) {
        const int r = SW * L.bsub + L.rho + zr, c = SW * (zh + 1 - L.bsub) + 4 * L.q;
        cp_async16_if(d, g, c >= 2 * SW && c < w && unsigned(y0 + r) < unsigned(h));
        cp_async16_if(d2, g2, c - 32 >= 2 * SW && c - 32 < w && unsigned(y0 + r + 32) < unsigned(h));
    } else {
        cp_async16f(d, g);
        cp_async16f(d2, g2);
    }
}

// The extra ring rows (alpha -K..-1 and 64, image -(K-1)..-1, F and B 64):
// one lane per 16-byte piece (lanes 0..4K+15), each with a static (plane,
// row, piece); in the group whose refill rows include its row it copies the
// row's next segment, with every check.
struct ExtraLane {
    const float* base;  // the piece's plane row (band row r), column 4 q
    unsigned sdst;      // its ring row, column 4 q (bytes)
    int r, m;           // band row; Z offset of its plane (mlo - phase)
    int q;
    bool on;
};

// (K = 4 has 40 extra pieces: slots 32..39 in a second instruction)
template <int K>
__device__ __forceinline__ constexpr bool extra2() { return 8 * K + 8 > 32; }

template <int K, int CK>
__device__ __forceinline__ ExtraLane make_extra(const RefillSrc& S, unsigned sbase, int slot) {
    using G = Geom<K, CK>;
    ExtraLane e;
    int p = 0;
    e.q = slot & 3;
    const int item = slot >> 2;  // alpha -K..-1: items 0..K-1; image -(K-1)..-1: K..2K-2; alpha/F/B 64: 2K-1..2K+1
    if (item < K) {
        p = 0;
        e.r = item - K;
    } else if (item < 2 * K - 1) {
        p = 1;
        e.r = item - K - (K - 1);
    } else {
        p = item - (2 * K - 1);  // 0 alpha, 1 -> F (2), 2 -> B (3)
        if (p > 0) ++p;
        e.r = BR;
    }
    e.on = item <= 2 * K + 1;
    if (!e.on) p = 0, e.r = 0;
    e.m = p == 0 ? G::mlo(0) - G::phase(0) : p == 1 ? G::mlo(1) - G::phase(1) : G::mlo(2) - G::phase(2);
    e.base = (p == 0 ? S.base[0] : p == 1 ? S.base[1] : p == 2 ? S.base[2] : S.base[3]) +
             (long long)e.r * (p <= 1 ? S.pitch[0] : S.pitch[2]) + 4 * e.q;
    const int lo = p == 0 ? G::LA : p == 1 ? G::LI : 0;
    const int off = p == 0 ? G::OFF_A : p == 1 ? G::OFF_I : p == 2 ? G::OFF_F : G::OFF_B;
    e.sdst = sbase + 4u * unsigned(off + (e.r - lo) * 32 + 4 * e.q);
    return e;
}

template <int K, int CK>
__device__ __forceinline__ void refill_extra(const ExtraLane& e, int t4, int y0, int w, int h) {
    const int Z = t4 + e.m;
    const int rr = e.r - (Z & 15);
    const int beta = rr >> 4;  // (arithmetic: rows above the block of Z)
    const int c = 16 * ((Z >> 4) + 1 - beta) + 4 * e.q;
    const bool ok = e.on && (rr & 15) < 4 && c >= 32 && c < w && unsigned(y0 + e.r) < unsigned(h);
    cp_async16_if(e.sdst + 4u * unsigned(c & 31) - 16u * e.q, e.base + (c - 4 * e.q), ok);
}

// Prologue: segments 0 and 1 of every ring row of plane P.
template <int K, bool V4, int CK, int P>
__device__ __forceinline__ void refill_prologue_p(const RefillSrc& S, unsigned sbase, int lane, int y0, int w, int h) {
    constexpr int PPR = plane_rw(P) / 4;  // pieces per ring row
    constexpr int N = plane_rows<K, CK>(P) * PPR;
    for (int it = lane; it < N; it += 32)
        put_piece<K, V4, CK, P>(S, sbase, it / PPR + plane_lo<K, CK>(P), 4 * (it % PPR), y0, w, h);
}
template <int K, bool V4, int CK>
__device__ __forceinline__ void refill_prologue(const RefillSrc& S, unsigned sbase, int lane, int y0, int w, int h) {
    refill_prologue_p<K, V4, CK, 0>(S, sbase, lane, y0, w, h);
    refill_prologue_p<K, V4, CK, 1>(S, sbase, lane, y0, w, h);
    refill_prologue_p<K, V4, CK, 2>(S, sbase, lane, y0, w, h);
    refill_prologue_p<K, V4, CK, 3>(S, sbase, lane, y0, w, h);
}

// ---- boundary-stream chunks ---------------------------------------------------
template <int K, int CK>
__device__ __forceinline__ bool chunk_complete(float4 q, int u0, int Umax, int lane) {
    using G = Geom<K, CK>;
    const int nvalid = min(CK, Umax - u0) * K * 2;  // floats
    const bool mine = lane < G::CH4 && 4 * lane < nvalid;
    if (!mine) return true;
    const int b = 4 * lane;
    return !(is_sentinel(q.x) || (b + 1 < nvalid && is_sentinel(q.y)) || (b + 2 < nvalid && is_sentinel(q.z)) ||
             (b + 3 < nvalid && is_sentinel(q.w)));
}

// The launch-wide failure state of a sweep: a per-launch abort flag (zeroed
// with the ticket) and a persistent per-device fault counter.
struct SweepFail {
    int* abort_flag;
    int* fault_count;
    unsigned long long spin_ns;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Poll chunk `u0 / CK` of the band above until every word of it is written;
// leaves it in the chunk buffer.  `v` holds a load issued earlier and is
// re-polled only while incomplete.  Bounded: after spin_ns the wait raises the
// launch's abort flag, counts a device fault and returns false; every other
// waiter of the launch then gives up at once.
template <int K, int CK>
__device__ __forceinline__ bool acquire_chunk(float4 v, const float* up_stream, int u0, int Umax, int lane,
                                              const SweepFail& F) {
    using G = Geom<K, CK>;
    const int nvalid = min(CK, Umax - u0) * K * 2;
    const bool mine = lane < G::CH4 && 4 * lane < nvalid;
    unsigned long long t0 = 0;
    for (unsigned n = 0; !__all_sync(kFull, chunk_complete<K, CK>(v, u0, Umax, lane)); ++n) {
        __nanosleep(32);
        if (mine) v = ld_relaxed_v4(up_stream + size_t(u0) * K * 2 + 4 * lane);
        if ((n & 255u) == 255u) {  // the abort flag and the clock every 256 polls
            int ab = 0;
            if (lane == 0) {
                const unsigned long long now = global_ns();
                if (!t0) t0 = now;
                ab = *reinterpret_cast<volatile int*>(F.abort_flag);
                if (!ab && now - t0 > F.spin_ns) {
                    atomicExch(F.abort_flag, 1);
                    atomicAdd(F.fault_count, 1);
                    ab = 1;
                }
            }
            if (__shfl_sync(kFull, ab, 0)) return false;
        }
    }
    if (mine) sts4(G::OFF_C + 4 * lane, v);
    return true;
}

template <int K, bool V4, int CK>
__device__ __forceinline__ void run_band(const SweepJob& J, int q, int ch, int lane, unsigned sbase, float eps,
                                         float omega, const SweepFail& F, int fault) {
    using G = Geom<K, CK>;
    const int w = J.w, h = J.h;
    const int y0 = q * BR;
    const int Umax = w + K - 1;
    const size_t slen = sweep_stream_len(w, K);
    const int sid = q * 3 + ch;
    const float* up_stream = q > 0 ? J.stream + size_t(sid - 3) * slen : nullptr;

    StepCtx cx;
    cx.lane = lane;
    cx.y0 = y0;
    cx.w = w;
    cx.h = h;
    cx.Umax = Umax;
    cx.lb4 = 256u * unsigned(lane);
    cx.ob4 = unsigned(4 * G::OFF_O + 8 * orow(2 * lane) * G::OW);
    cx.flb4 = unsigned(4 * G::OFF_O + 8 * (17 * (lane >> 4) * G::OW + (lane & 15)));
    cx.has_up = q > 0;
    cx.has_down = q < J.nb - 1 && !(fault == 1 && q == 0);  // (fault 1: band 0 never publishes)
    cx.my_stream = J.stream + size_t(sid) * slen;
    {
        const long long fo = (long long)(y0 - (K - 1)) * J.opitch + 16LL * (lane >> 4) * (J.opitch - 1) +
                             (lane & 15) - K - 14;
        cx.gF = J.fg_out + (long long)ch * J.ostride + fo;
        cx.gB = J.bg_out + (long long)ch * J.ostride + fo;
    }
    cx.op1 = J.opitch - 1;
    cx.ytop = cx.ybot = 0;
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int y = y0 + 2 * lane + i - k;
            if (y <= 0) cx.ytop |= 1u << (i * K + k);
            if (y >= h - 1) cx.ybot |= 1u << (i * K + k);
        }
    cx.eps = eps;
    cx.omega = omega;

    RefillSrc S;
    S.base[0] = J.alpha + (long long)y0 * J.ipitch;
    S.base[1] = J.img + (long long)ch * J.istride + (long long)y0 * J.ipitch;
    S.base[2] = J.fg_in + (long long)ch * J.fstride + (long long)y0 * J.fpitch;
    S.base[3] = J.bg_in + (long long)ch * J.fstride + (long long)y0 * J.fpitch;
    S.pitch[0] = S.pitch[1] = J.ipitch;
    S.pitch[2] = S.pitch[3] = J.fpitch;
    // this lane's piece of the main refill blocks: rows SW bsub + rho (+ Z mod
    // SW; + 32 for the second instruction), columns SW (1 - bsub) + 4 q
    // (+ SW (Z div SW))
    int gl[4];
    unsigned ssl[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int SW = 16, PPS = SW / 4;
        const int q = lane % PPS, rho = (lane / PPS) & 3, bsub = lane / (4 * PPS);
        gl[p] = (SW * bsub + rho) * S.pitch[p] + SW * (1 - bsub) + 4 * q;
        ssl[p] = sbase + 4u * unsigned((SW * bsub + rho) * 2 * SW + 4 * q);
    }
    const ExtraLane xtra = make_extra<K, CK>(S, sbase, lane);
    const ExtraLane xtra2 = make_extra<K, CK>(S, sbase, lane + 32);
    refill_prologue<K, V4, CK>(S, sbase, lane, y0, w, h);
    cp_commit();
    cp_commit();  // (an empty group: the first wait_group<1> covers the prologue)

    LaneState<K> st;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        st.o[0][k] = st.o[1][k] = st.o2[k] = st.rvp[k] = make_float2(0.0f, 0.0f);
        st.cp1[k] = st.cp2[k] = coef_w(0.5f, 1.0f, 1.0f, 1.0f, 1.0f, 0.0f);
        st.dRr[k] = eps;
    }
    st.aRp[0] = st.aRp[1] = st.aU0p = st.a0p = 0.0f;
    st.FRp[0] = st.FRp[1] = make_float2(0.0f, 0.0f);
    st.dRp[0] = st.dRp[1] = st.dDp = eps;

    float4 pend = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool lane_ch = lane < G::CH4;
    bool pend_ok = false;  // pend holds the complete next chunk
    if (cx.has_up && lane_ch) pend = ld_relaxed_v4(up_stream + 4 * lane);

    const bool yband = y0 - (K - 1) <= 0 || y0 + BR - 1 >= h - 1;
    // Steps t4..t4+3 have every pixel at 1 <= x <= w - 2, every flushed
    // segment at x >= 0 and every stream slot in range iff
    // t4 >= fast_lo (t4 - 63 - (K-1) >= 1 and t4 - K - 14 - 63 >= 0) and
    // t4 + 3 <= fast_hi.  Left-region groups (t4 < fast_lo) need no right
    // checks when fast_lo + 3 <= fast_hi.
    const int fast_lo = (78 + K + 3) & ~3, fast_hi = w - 2;
    const bool split = fast_lo + 3 <= fast_hi;
    // refills of groups t4 in [rf_lo, rf_hi) are inside rows 0..63 and [32, w)
    const bool rf_band = J.vec4 && y0 >= K && y0 + BR < h;
    const int rf_lo = 72 + 2 * K, rf_hi = w - 32;
    const int tend = Umax + BR - 1;  // steps t < tend
    for (int t4 = -4; t4 < tend; t4 += 4) {
        cp_wait<G::WAITN>();
        __syncwarp();
        if (cx.has_up && t4 >= 0 && t4 < Umax) {
            const int nxt = (t4 & ~(CK - 1)) + CK;  // the next chunk's first column
            if ((t4 & (CK - 1)) == 0) {
                if (!acquire_chunk<K, CK>(pend, up_stream, t4, Umax, lane, F)) {
                    cp_wait<0>();  // the launch is aborted: drop the band
                    __syncwarp();
                    return;
                }
                pend_ok = false;
                if (nxt < Umax && lane_ch) pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
            } else if (!pend_ok && nxt < Umax) {
                // the prefetch found the next chunk incomplete: re-poll it now
                pend_ok = __all_sync(kFull, chunk_complete<K, CK>(pend, nxt, Umax, lane));
                if (!pend_ok && lane_ch) pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
            }
            __syncwarp();
        }
        const int c4g = 4 * t4 - 8 * lane;
        const bool xl = t4 < fast_lo, xr = t4 + 3 > fast_hi;
        if (!xl && !xr && !yband) {
#pragma unroll
            for (int s = 0; s < 4; ++s) band_step<K, CK, 0, false>(st, cx, c4g, t4, s);
        } else if (!xl && !xr) {
#ifdef FGM_Y_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
            for (int s = 0; s < 4; ++s) band_step<K, CK, 0, true>(st, cx, c4g, t4, s);
        } else if (split && !xr && !yband) {
#pragma unroll 1
            for (int s = 0; s < 4; ++s) band_step<K, CK, 1, false>(st, cx, c4g, t4, s);
        } else if (split && !xl && !yband) {
#pragma unroll 1
            for (int s = 0; s < 4; ++s) band_step<K, CK, 2, false>(st, cx, c4g, t4, s);
        } else if (split && !xr) {
#pragma unroll 1
            for (int s = 0; s < 4; ++s) band_step<K, CK, 1, true>(st, cx, c4g, t4, s);
        } else if (split && !xl) {
#pragma unroll 1
            for (int s = 0; s < 4; ++s) band_step<K, CK, 2, true>(st, cx, c4g, t4, s);
        } else {
#pragma unroll 1
            for (int s = 0; s < 4; ++s) band_step<K, CK, 3, true>(st, cx, c4g, t4, s);
        }
        __syncwarp();  // every lane is done with the ring slots the refills overwrite
        if (rf_band && t4 >= rf_lo && t4 < rf_hi) {
            refill_main_p<K, CK, 0, false>(S, gl[0], ssl[0], t4, lane, y0, w, h);
            refill_main_p<K, CK, 1, false>(S, gl[1], ssl[1], t4, lane, y0, w, h);
            refill_main_p<K, CK, 2, false>(S, gl[2], ssl[2], t4, lane, y0, w, h);
            refill_main_p<K, CK, 3, false>(S, gl[3], ssl[3], t4, lane, y0, w, h);
            refill_extra<K, CK>(xtra, t4, y0, w, h);
            if (extra2<K>()) refill_extra<K, CK>(xtra2, t4, y0, w, h);
        } else if (V4) {
            refill_main_p<K, CK, 0, true>(S, gl[0], ssl[0], t4, lane, y0, w, h);
            refill_main_p<K, CK, 1, true>(S, gl[1], ssl[1], t4, lane, y0, w, h);
            refill_main_p<K, CK, 2, true>(S, gl[2], ssl[2], t4, lane, y0, w, h);
            refill_main_p<K, CK, 3, true>(S, gl[3], ssl[3], t4, lane, y0, w, h);
            refill_extra<K, CK>(xtra, t4, y0, w, h);
            if (extra2<K>()) refill_extra<K, CK>(xtra2, t4, y0, w, h);
        } else {
            refill_checked<K, false, CK>(S, sbase, t4, lane, y0, w, h);
        }
        cp_commit();
    }
    cp_wait<0>();
    __syncwarp();
}

struct SweepArgs {
    const SweepJob* jobs;
    const int2* order;  // (job, band * 3 + channel) per ticket
    int total;
    unsigned* ticket;
    float eps, omega;
    SweepFail fail;
    int fault;  // debug fault injection (fgm_debug_fault)
};

template <int K, int CK>
__global__ void __launch_bounds__(32, 1) sweep_kernel(SweepArgs A) {
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sweep_sm4));
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned tk = 0;
        if (lane == 0) tk = atomicAdd(A.ticket, 1u);
        tk = __shfl_sync(kFull, tk, 0);
        if (tk >= unsigned(A.total) || *reinterpret_cast<volatile int*>(A.fail.abort_flag)) return;
        const int2 jb = A.order[tk];  // (job, band * 3 + channel)
        const SweepJob J = A.jobs[jb.x];
        if (J.vec4)
            run_band<K, true, CK>(J, jb.y / 3, jb.y % 3, lane, sbase, A.eps, A.omega, A.fail, A.fault);
        else
            run_band<K, false, CK>(J, jb.y / 3, jb.y % 3, lane, sbase, A.eps, A.omega, A.fail, A.fault);
    }
}

// Per-device launch state: the function attributes (both chunk widths) and
// the resident-warp capacity.
template <int K>
cudaError_t sweep_grid_cap(int& cap) {
    static PerDevice<int> cfg;
    return cfg.get(cap, [](int dev, int& v) {
        const int sm4 = int(Geom<K, 4>::TOTAL * sizeof(float)), sm16 = int(Geom<K, kChunk>::TOTAL * sizeof(float));
        cudaError_t e = cudaFuncSetAttribute(sweep_kernel<K, kChunk>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm16);
        // the largest shared-memory carveout: the rings, not L1, bound the resident warps
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_kernel<K, kChunk>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_kernel<K, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_kernel<K, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int sms = 0, per_sm = 0;
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<K, kChunk>, 32, size_t(sm16));
        v = std::max(1, sms * std::max(1, per_sm));
        return e;
    });
}

// Launches whose (band, channel) items all fit on the GPU at once are
// latency-bound single images: their critical path crosses every band, one
// boundary-stream chunk per hand-over, so they poll 4-column chunks (a shorter
// hand-over lag); throughput launches poll 16-column chunks.
template <int K>
cudaError_t launch_sweep_k(const SweepArgs& A, cudaStream_t s) {
    int cap = 0;
    cudaError_t e = sweep_grid_cap<K>(cap);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(A.total, cap));
    if (A.total <= cap)
        sweep_kernel<K, 4><<<grid, 32, size_t(Geom<K, 4>::TOTAL) * sizeof(float), s>>>(A);
    else
        sweep_kernel<K, kChunk><<<grid, 32, size_t(Geom<K, kChunk>::TOTAL) * sizeof(float), s>>>(A);
    return cudaGetLastError();
}

__global__ void stream_fill_kernel(const SweepJob* __restrict__ jobs, int K) {
    const SweepJob J = jobs[blockIdx.y];
    const size_t n = size_t(J.nb) * 3 * sweep_stream_len(J.w, K) / 4;
    float4* p = reinterpret_cast<float4*>(J.stream);
    const float s = __uint_as_float(kStreamSentinel);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = make_float4(s, s, s, s);
}

}  // namespace

cudaError_t launch_stream_fill(const SweepJob* jobs, int njobs, int K, size_t max_floats, cudaStream_t s) {
    if (njobs <= 0) return cudaSuccess;
    const int gx = int(std::min<size_t>(std::max<size_t>((max_floats / 4 + 255) / 256, 1), 64));
    stream_fill_kernel<<<dim3(gx, njobs), 256, 0, s>>>(jobs, K);
    return cudaGetLastError();
}

int sweep_supported_k(int K) { return K >= 1 && K <= 4; }

size_t sweep_smem_bytes(int K) {
    switch (K) {
        case 1: return Geom<1, kChunk>::TOTAL * sizeof(float);
        case 2: return Geom<2, kChunk>::TOTAL * sizeof(float);
        case 3: return Geom<3, kChunk>::TOTAL * sizeof(float);
        case 4: return Geom<4, kChunk>::TOTAL * sizeof(float);
        default: return 0;
    }
}

std::atomic<int> g_sweep_fault{0};
std::atomic<long long> g_spin_timeout_ns{2000000000ll};

cudaError_t launch_sweep(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket,
                         float eps, float omega, int* abort_flag, int* fault_count, cudaStream_t s) {
    SweepArgs A;
    A.jobs = jobs_dev;
    A.order = order_dev;
    A.total = total_items;
    A.ticket = ticket;
    A.eps = eps;
    A.omega = omega;
    A.fail.abort_flag = abort_flag;
    A.fail.fault_count = fault_count;
    A.fail.spin_ns = (unsigned long long)std::max<long long>(g_spin_timeout_ns.load(), 1000);
    A.fault = g_sweep_fault.load();
    switch (K) {
        case 1: return launch_sweep_k<1>(A, s);
        case 2: return launch_sweep_k<2>(A, s);
        case 3: return launch_sweep_k<3>(A, s);
        case 4: return launch_sweep_k<4>(A, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fgm
