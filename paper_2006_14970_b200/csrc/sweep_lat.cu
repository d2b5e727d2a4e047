// K3, latency path: the round-1 sweep kernel, one 32-row band per warp (one
// row per lane), chosen for launches of a few images, whose time is the
// wavefront's dependency chain (w + h steps of one lane) rather than
// throughput: a step of one row per lane has half the instructions of the
// two-row step of the throughput kernel (sweep.cu), so a lone band steps
// faster.  Batches use sweep.cu.
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
// one chunk ahead and re-polled once per group while incomplete.
//
// The three colour channels share only alpha (the 2x2 matrix is common to all
// channels, multilevel.hpp:37-43), so each (band, channel) is an independent
// warp: it computes the alpha-only coefficients of its pixels and runs the
// F_c / B_c recurrence (pixel_apply1) of its channel.  The left edge weight
// of a pixel is the right edge weight of the pixel the same slot updated one
// step earlier (|a - b| is exactly symmetric), so only three are computed.
//
// Memory: each warp streams its band's rows of alpha, I_c and the initial F_c,
// B_c through per-row shared-memory rings of 32 columns, filled by cp.async
// 16-byte blocks M groups ahead of use.  Element (row r, column x) sits at
// ring column x mod 32; the first MIR columns are mirrored after column 31, so
// every read of a step is  lane_base + 4*c + (compile-time offset)  with one
// c = (t - lane - SH) mod 32 per step -- no per-access index arithmetic.  Rows
// are RS = 32 + MIR floats apart: the diagonal reads of a step hit banks
// (RS - 1) * lane + const, all distinct since RS - 1 is odd.  Outputs go
// through a 16-column ring per row and leave as 64-byte row segments (two
// rows per step) once complete.  Steps run in groups of four: loads, stream
// chunks and the border/fast decision are handled once per group.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "fgm_device.cuh"
#include "fgm_internal.h"

namespace fgm {
namespace {

constexpr int kLatRows = 32;  // band rows (one per lane)

__device__ __forceinline__ void cp_async16(unsigned sdst, const float* gsrc, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sdst), "l"(gsrc), "r"(src_bytes) : "memory");
}
// Predicated 16-byte copy without zero-fill (a predicate, not a branch).
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
// Boundary-stream stores need no ordering against this warp's other memory
// operations (every word validates itself), hence no "memory" clobber: the
// compiler may keep scheduling shared-memory loads across them.
__device__ __forceinline__ void st_relaxed_v4(float* p, float4 v) {
    asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
}
__device__ __forceinline__ void st_relaxed_v2(float* p, float2 v) {
    asm volatile("st.relaxed.gpu.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y));
}
// The dynamic shared memory of the sweep kernel, addressed by float index:
// the compiler sees shared-space accesses (LDS/STS with the compile-time part
// of an index folded into the instruction) and orders them against
// __syncwarp and the cp.async waits.
extern __shared__ float4 sweep_sm4[];
__device__ __forceinline__ float* smf() { return reinterpret_cast<float*>(sweep_sm4); }
__device__ __forceinline__ float lds(int i) { return smf()[i]; }
__device__ __forceinline__ void sts(int i, float v) { smf()[i] = v; }
__device__ __forceinline__ void sts4(int i, float4 v) { reinterpret_cast<float4*>(smf() + i)[0] = v; }
__device__ __forceinline__ void stg(float* p, float v) { __stcg(p, v); }
__device__ __forceinline__ bool is_sentinel(float v) { return __float_as_uint(v) == kStreamSentinel; }
#ifndef FGM_GROUP
#define FGM_GROUP 4
#endif
// Shared-memory geometry of one (band, channel) warp, in floats.
//
// Ring window.  In row-time tau = x + r (band row r, column x) the reads of
// step t cover alpha tau in [t-2K+2, t+2] (the next step's pixels and their
// four neighbours), image [t-2K+3, t+1] and the initial F/B [t, t+1].  Steps
// run in groups of S = 4; the S-column blocks of every row are issued at
// the end of each group with a lead L = S*M - 1 + W1 (W1 = the window's reach
// past the group), so a group waits only for loads issued M groups earlier;
// the live span S*M + S - 1 + W0 + W1 must fit in the 32 ring columns
// (static_asserts below).
template <int K, int CK = kChunk>
struct Geom {
    static constexpr int RW = 32;               // ring columns
    static constexpr int SH = K - 1;            // read column shift: offsets d + SH >= 0
    static constexpr int MIR = K <= 2 ? 4 : 8;  // mirrored columns (> largest shifted offset)
    static constexpr int RS = RW + MIR;         // row stride (floats), 16-byte multiple, RS - 1 odd
    // steps per group = columns per load block.  (8 in throughput launches
    // runs 2% fewer instructions but measured 3% slower on the C4 batch: the
    // four unrolled 8-step paths no longer share the instruction cache.)
    static constexpr int S = FGM_GROUP;
    static constexpr int M = 16 / S;            // load groups in flight
    static constexpr int L = S * M + 1;         // load lead: S*M - 1 + W1, W1 = 2 (alpha; 1 for the others)
    static constexpr int NA = 33 + K;           // alpha ring rows: band rows -K .. 32
    static constexpr int NI = 31 + K;           // image ring rows: band rows -(K-1) .. 31
    static constexpr int NF = 33;               // F/B ring rows: band rows 0 .. 32
    static constexpr int OW = 16;               // output ring columns
    static constexpr int OFF_A = 0;
    static constexpr int OFF_I = OFF_A + NA * RS;
    static constexpr int OFF_F = OFF_I + NI * RS;
    static constexpr int OFF_B = OFF_F + NF * RS;
    static constexpr int OFF_O = OFF_B + NF * RS;  // [plane F/B][orow(j)][OW]
    static constexpr int OPL = 33 * OW;
    static constexpr int OFF_C = OFF_O + 2 * OPL;
    static constexpr int CH = CK * K * 2;      // one boundary-stream chunk of CK columns: [u][k][F,B]
    static constexpr int CH4 = CH / 4;         // float4 per chunk (<= 32: one per lane)
    static constexpr int TOTAL = OFF_C + CH;
    static_assert(L + (2 * K - 2) + S <= RW, "alpha ring too small for its lead");
    static_assert(2 + SH <= MIR && MIR % 4 == 0 && RS % 4 == 0, "mirror too narrow");
    static_assert(CH % 4 == 0 && CH4 <= 32, "a chunk is at most one float4 per lane");
};

// output ring row of band row j (a padding row after row 15: the diagonal
// writes and the two-row flush reads hit distinct banks)
__device__ __forceinline__ constexpr int orow(int j) { return j + (j >> 4); }

// The global rows a lane streams into its rings (its own row and, for some
// lanes, one extra row: alpha -K..-1 and 32, image -(K-1)..-1, F/B 32).
// Ring rows of one band row sit at compile-time offsets from `s` (alpha row
// r + K, image row r + K - 1, F/B row r); planes the lane does not stream, or
// rows outside the image, are masked off in `vm` (their ring slots are never
// read unclamped).
struct RowSrc {
    const float* g[4];  // alpha, image c, F_c, B_c rows (column 0)
    unsigned s;         // shared address of ring offset 0, ring row r, column 0
    unsigned vm;        // bit p: plane p is streamed
    int r;              // row relative to the band
};

template <int K>
__device__ __forceinline__ RowSrc make_rowsrc(const SweepJob& J, int ch, int y0, int r, bool doA, bool doI, bool doF,
                                              unsigned sbase) {
    using G = Geom<K>;
    RowSrc rs;
    const int y = y0 + r;
    const bool ok = y >= 0 && y < J.h;
    const long long oi = (long long)(ok ? y : 0) * J.ipitch, of = (long long)(ok ? y : 0) * J.fpitch;
    rs.g[0] = J.alpha + oi;
    rs.g[1] = J.img + ch * J.istride + oi;
    rs.g[2] = J.fg_in + ch * J.fstride + of;
    rs.g[3] = J.bg_in + ch * J.fstride + of;
    rs.s = sbase + 4u * unsigned(r * G::RS);  // may wrap below sbase: only ever offset back into range
    rs.vm = ok ? (doA ? 1u : 0u) | (doI ? 2u : 0u) | (doF ? 12u : 0u) : 0u;
    rs.r = r;
    return rs;
}

// Ring offset (floats) of plane p's row r relative to ring row r of offset 0.
template <int K>
__device__ __forceinline__ constexpr int plane_off(int p) {
    using G = Geom<K>;
    return p == 0 ? G::OFF_A + K * G::RS : p == 1 ? G::OFF_I + (K - 1) * G::RS : p == 2 ? G::OFF_F : G::OFF_B;
}

// cp.async of the S-column block at column x0 (S-aligned) of every streamed
// plane of one row into the rings, as 4-column pieces (each also into the
// mirror columns when it lands in the first MIR columns).  Columns past the
// row end are zero-filled (src-size); pieces outside [0, w) are skipped.
template <int K, bool V4, int CK>
__device__ __forceinline__ void put_blocks(const RowSrc& rs, int x0, int w) {
    using G = Geom<K, CK>;
    if (x0 < 0) return;
#pragma unroll
    for (int b = 0; b < G::S / 4; ++b) {
        const int xb = x0 + 4 * b;
        if (xb >= w) return;
        const int nb = min(w - xb, 4) * 4;
        const int c = xb & (G::RW - 1);
        const unsigned sc = rs.s + 4u * c;
        const bool mir = c < G::MIR;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            if (!(rs.vm & (1u << p))) continue;
            const float* g = rs.g[p] + xb;
            const unsigned d = sc + 4u * plane_off<K>(p);
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
}

// The block of one row issued at the end of group t4 (lead L).
template <int K, bool V4, int CK>
__device__ __forceinline__ void issue_row(const RowSrc& rs, int t4, int w) {
    using G = Geom<K, CK>;
    put_blocks<K, V4, CK>(rs, (t4 + G::S + G::L - rs.r) & ~(G::S - 1), w);
}

// Interior groups of 16-byte-aligned jobs: every lane's block is inside
// [0, w), so no range checks and no zero-fill; the per-lane plane mask and
// the mirror copy become instruction predicates.  MASK: compile-time plane
// mask (15 for a lane's own row of an interior band), else rs.vm.
template <int K, unsigned MASK, int CK>
__device__ __forceinline__ void issue_row_fast(const RowSrc& rs, int t4) {
    using G = Geom<K, CK>;
    const unsigned x0 = unsigned(t4 + G::S + G::L - rs.r) & ~unsigned(G::S - 1);  // >= 0 in interior groups
    const unsigned c = x0 & (G::RW - 1);  // S-aligned: the pieces of a block never wrap the ring
    const unsigned sc = rs.s + 4u * c;
    const unsigned vm = MASK ? MASK : rs.vm;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const float* g = rs.g[p] + x0;
        const unsigned d = sc + 4u * plane_off<K>(p);
        const unsigned on = (vm >> p) & 1u;
#pragma unroll
        for (int b = 0; b < G::S / 4; ++b) {
            cp_async16_if(d + 16u * b, g + 4 * b, on);
            if (4 * b < G::MIR)  // only the first MIR columns of the ring are mirrored
                cp_async16_if(d + 16u * b + 4u * G::RW, g + 4 * b, on & (c + 4u * b < unsigned(G::MIR) ? 1u : 0u));
        }
    }
}

// Interior groups of interior bands, flattened: the 130 + 2K (plane, band
// row) blocks a group issues (alpha rows -K..32, image rows -(K-1)..31, F and
// B rows 0..32) are dealt to the lanes of ceil((130 + 2K) / 32) cp.async
// instructions instead of one own-row and one extra-row instruction per plane
// (the extra rows occupy three lanes).  Per lane and instruction: the row's
// global base, its ring address and its lead q = S + L - r, all fixed per band.
template <int K>
struct FlatSrc {
    static constexpr int N = (130 + 2 * K + 31) / 32;
    const float* g[N];
    unsigned s[N];
    int q[N];
    unsigned on;  // bit i: lane holds an item in instruction i
};

template <int K, int CK>
__device__ __forceinline__ FlatSrc<K> make_flat(const SweepJob& J, int ch, int y0, int lane, unsigned sbase) {
    using G = Geom<K, CK>;
    FlatSrc<K> f;
    f.on = 0;
    constexpr int NAl = 33 + K, NIm = 31 + K, NFB = 33;
#pragma unroll
    for (int i = 0; i < FlatSrc<K>::N; ++i) {
        int it = 32 * i + lane;
        int p = 0, r = 0;
        if (it < NAl) {
            p = 0;
            r = it - K;
        } else if ((it -= NAl) < NIm) {
            p = 1;
            r = it - (K - 1);
        } else if ((it -= NIm) < NFB) {
            p = 2;
            r = it;
        } else if ((it -= NFB) < NFB) {
            p = 3;
            r = it;
        } else {
            p = -1;
        }
        const int y = min(max(y0 + r, 0), J.h - 1);  // (in range for interior bands)
        const float* base = p == 0 ? J.alpha + (long long)y * J.ipitch
                          : p == 1 ? J.img + ch * J.istride + (long long)y * J.ipitch
                          : p == 2 ? J.fg_in + ch * J.fstride + (long long)y * J.fpitch
                                   : J.bg_in + ch * J.fstride + (long long)y * J.fpitch;
        f.g[i] = base;
        const int po = p == 0 ? plane_off<K>(0) : p == 1 ? plane_off<K>(1) : p == 2 ? plane_off<K>(2) : plane_off<K>(3);
        f.s[i] = sbase + 4u * unsigned(po + r * G::RS);
        f.q[i] = G::S + G::L - r;
        if (p >= 0) f.on |= 1u << i;
    }
    return f;
}

template <int K, int CK>
__device__ __forceinline__ void issue_flat(const FlatSrc<K>& f, int t4) {
    using G = Geom<K, CK>;
#pragma unroll
    for (int i = 0; i < FlatSrc<K>::N; ++i) {
        const unsigned x0 = unsigned(t4 + f.q[i]) & ~unsigned(G::S - 1);
        const unsigned c = x0 & (G::RW - 1);
        const float* g = f.g[i] + x0;
        const unsigned d = f.s[i] + 4u * c;
        const unsigned on = (f.on >> i) & 1u;
#pragma unroll
        for (int b = 0; b < G::S / 4; ++b) {
            cp_async16_if(d + 16u * b, g + 4 * b, on);
            if (4 * b < G::MIR)
                cp_async16_if(d + 16u * b + 4u * G::RW, g + 4 * b, on & (c + 4u * b < unsigned(G::MIR) ? 1u : 0u));
        }
    }
}

// Everything issued "before group t0".
template <int K, bool V4, int CK>
__device__ __forceinline__ void prologue_row(const RowSrc& rs, int t0, int w) {
    using G = Geom<K, CK>;
    const int last = (t0 + G::L - rs.r) & ~(G::S - 1);  // the block issued at the end of group t0 - S
    for (int x0 = 0; x0 <= last; x0 += G::S) put_blocks<K, V4, CK>(rs, x0, w);
}

// Packed (F, B) arithmetic (FFMA2, fgm_device.cuh) or the scalar form; the
// two are bitwise identical.
#ifndef FGM_PACKED
#define FGM_PACKED 2
#endif
#if FGM_PACKED == 2
using SCoef = CoefR;
__device__ __forceinline__ SCoef coef_dl(float a, float dL, float aR, float aU, float aD, float I, float eps,
                                         float omega) {
    return pixel_coefr_dl(a, dL, aR, aU, aD, I, eps, omega);
}
__device__ __forceinline__ float2 apply_coef(const SCoef& co, float2 L, float2 R, float2 U, float2 D) {
    return pixel_applyr(co, L, R, U, D);
}
#elif FGM_PACKED
using SCoef = CoefP;
__device__ __forceinline__ SCoef coef_dl(float a, float dL, float aR, float aU, float aD, float I, float eps,
                                         float omega) {
    return pixel_coefp_dl(a, dL, aR, aU, aD, I, eps, omega);
}
__device__ __forceinline__ float2 apply_coef(const SCoef& co, float2 L, float2 R, float2 U, float2 D) {
    return pixel_applyp(co, L, R, U, D);
}
#else
using SCoef = Coef1;
__device__ __forceinline__ SCoef coef_dl(float a, float dL, float aR, float aU, float aD, float I, float eps,
                                         float omega) {
    return pixel_coef1_dl(a, dL, aR, aU, aD, I, eps, omega);
}
__device__ __forceinline__ float2 apply_coef(const SCoef& co, float2 L, float2 R, float2 U, float2 D) {
    return pixel_apply1(co, L, R, U, D);
}
#endif

// Float offset, from rc = lane_base + c, of ring `off`, ring row lane + row,
// shifted column offset dp.
template <int K>
__device__ __forceinline__ constexpr int ring(int off, int row, int dp) {
    return off + row * Geom<K>::RS + dp;
}

// Coefficients of slot k's pixel of the next step (column offset 1 - k from
// t - lane), its left edge weight `dL` given.  G: clamp neighbours at the
// image border.
template <int K, bool G, bool Y = false, bool XL = false>
__device__ __forceinline__ SCoef next_coef(int rc, int k, float dL, int x, int y, int w, int h, float eps,
                                           float omega) {
    using Gm = Geom<K>;
    const int dp = 1 - k + Gm::SH;  // shifted column of the pixel
    const int ar = K - k;           // alpha ring row (relative to lane) of the pixel
    const float a = lds(rc + ring<K>(Gm::OFF_A, ar, dp));
    float aR = lds(rc + ring<K>(Gm::OFF_A, ar, dp + 1));
    float aU = lds(rc + ring<K>(Gm::OFF_A, ar - 1, dp));
    float aD = lds(rc + ring<K>(Gm::OFF_A, ar + 1, dp));
    const float I = lds(rc + ring<K>(Gm::OFF_I, K - 1 - k, dp));
    if (G || XL) {
        if (x <= 0) dL = eps;  // edge_weight(a, a)
    }
    if (G) {
        if (x >= w - 1) aR = a;
    }
    if (G || Y) {
        if (y <= 0) aU = a;
        if (y >= h - 1) aD = a;
    }
    return coef_dl(a, dL, aR, aU, aD, I, eps, omega);
}

// Coefficients from scratch (the first step of a band: no left pixel yet).
template <int K>
__device__ __forceinline__ SCoef first_coef(int rc, int k, int x, int y, int w, int h, float eps, float omega) {
    using Gm = Geom<K>;
    const int dp = 1 - k + Gm::SH;
    const int ar = K - k;
    const float a = lds(rc + ring<K>(Gm::OFF_A, ar, dp));
    const float aL = lds(rc + ring<K>(Gm::OFF_A, ar, dp - 1));
    const float dL = edge_weight(a, x <= 0 ? a : aL, eps, omega);
    return next_coef<K, true>(rc, k, dL, x, y, w, h, eps, omega);
}

template <int K>
struct LaneState {
    float2 outp[K];   // this lane's (F_c, B_c) outputs of the previous step
    float2 rprev[K];  // what this lane received from lane-1 at the previous step (border steps)
    SCoef co[K];      // coefficients of this step's pixels (computed one step ahead)
};

template <int K>
struct StepCtx {
    int lb;  // float index of ring offset 0, row "lane", column 0
    int ob;  // output ring row orow(lane), column 0
    int lane, y0, w, h;
    bool has_up, has_down;
    int Umax;
    float* my_stream;  // this band's stream (column 0)
    float* FO;  // output planes at band row 0 (image row y0 - (K-1))
    float* BO;
    int opitch;
    float eps, omega;
};

// One wavefront step.  G: a pixel of this step or the next may be on the
// image border (clamped neighbours) or an output row segment may be partial.
// Y (with G false): interior columns of a band touching row 0 or h-1: only
// the row clamps and the output row bounds of G (the first band heads every
// image's chain, so it must not run at border-path speed).
// XL (with G false): the first steps of a band, where only the left column
// border occurs (x <= 0): the L clamp and the bounds of the stream and the
// flush, as selects and predicates.  Every band's start is on the chain's
// critical path (the band below waits for it).
// Per-group addressing of the interior paths.  With K = 2 (mod 4) a group's
// four flushed output rows never cross a 16-row half of the output ring
// (u = t - (K-1) - 15 starts the group at a multiple of 4), so step s of the
// group flushes row jf0 + s of segment xs0: the global addresses advance by
// one output row per step and the ring offsets by one ring row, and lane 31's
// boundary-stream slot by 2K floats (an immediate offset).
template <int K>
struct GroupAddr {
    float* fo;        // flush address of step 0, F plane
    float* bo;        // and B plane
    int o0;           // output-ring float index of step 0
    bool seg_ok;      // XL: the segment start column is inside the row
    int jf0;          // flushed band row of step 0
    float* sdst;      // lane 31's boundary-stream slot of step 0
};
template <int K>
__device__ __forceinline__ constexpr bool group_addr_ok() { return K % 4 == 2; }

template <int K, int CK>
__device__ __forceinline__ GroupAddr<K> group_addr(const StepCtx<K>& x_, int t4) {
    using Gm = Geom<K, CK>;
    constexpr int OW = Gm::OW;
    GroupAddr<K> g;
    const int lane = x_.lane;
    const int col = lane & (OW - 1);
    const int u0 = t4 - (K - 1) - (OW - 1);
    g.jf0 = (u0 & (OW - 1)) + (lane & 16);
    const int xs0 = (u0 & ~(OW - 1)) - (lane & 16);
    g.seg_ok = xs0 >= 0;
    const unsigned off = unsigned(g.jf0 * x_.opitch + xs0 + col);  // (used only when seg_ok)
    g.fo = x_.FO + off;
    g.bo = x_.BO + off;
    g.o0 = Gm::OFF_O + orow(g.jf0) * OW + col;
    g.sdst = x_.my_stream + (long long)(t4 - 31) * K * 2;
    return g;
}

template <int K, bool G, int CK, bool Y = false, bool XL = false>
__device__ __forceinline__ void band_step(LaneState<K>& st, const StepCtx<K>& x_, int tr,
                                          const GroupAddr<K>* ga = nullptr, int gs = 0) {
    using Gm = Geom<K, CK>;
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
        const int cn = Gm::OFF_C + (tr % CK) * K * 2;
#pragma unroll
        for (int k = 0; k < K; ++k) recv[k] = make_float2(lds(cn + 2 * k), lds(cn + 2 * k + 1));
    }

    float2 nv[K];
    const int xs0 = tr - lane;  // slot-0 column
#pragma unroll
    for (int k = 0; k < K; ++k) {
        float2 L = st.outp[k], U = recv[k], R, D;
        if (k == 0) {
            R = make_float2(lds(rc + ring<K>(Gm::OFF_F, 0, 1 + Gm::SH)), lds(rc + ring<K>(Gm::OFF_B, 0, 1 + Gm::SH)));
            D = make_float2(lds(rc + ring<K>(Gm::OFF_F, 1, Gm::SH)), lds(rc + ring<K>(Gm::OFF_B, 1, Gm::SH)));
        } else {
            R = recv[k - 1];
            D = st.outp[k - 1];
        }
        if (G || Y || XL) {
            const int x = xs0 - k, y = y0 + lane - k;
            const float2 self = k == 0 ? make_float2(lds(rc + ring<K>(Gm::OFF_F, 0, Gm::SH)),
                                                     lds(rc + ring<K>(Gm::OFF_B, 0, Gm::SH)))
                                       : st.rprev[k > 0 ? k - 1 : 0];
            if (G || XL) {
                if (!(x > 0)) L = self;
            }
            if (G) {
                if (!(x < w - 1)) R = self;
            }
            if (G || Y) {
                if (!(y > 0)) U = self;
                if (!(y < h - 1)) D = self;
            }
        }
        nv[k] = apply_coef(st.co[k], L, R, U, D);
    }

    // coefficients of the next step's pixels; dL = this step's dR of the slot
#pragma unroll
    for (int k = 0; k < K; ++k)
        st.co[k] = next_coef<K, G, Y, XL>(rc, k, st.co[k].dR, xs0 + 1 - k, y0 + lane - k, w, h, x_.eps, x_.omega);

    // output ring (last sweep only): column x & 15 == c & 15
    {
        bool ok = true;
        if (G) {
            const int x = xs0 - (K - 1);
            ok = x >= 0 && x < w && y0 + lane - (K - 1) >= 0 && y0 + lane - (K - 1) < h;
        }
        if (ok) {  // (Y: rows outside the image land in the ring but are never flushed)
            const int o = x_.ob + (c & (OW - 1));
            sts(o, nv[K - 1].x);
            sts(o + Gm::OPL, nv[K - 1].y);
        }
    }

    // boundary stream for the band below: lane 31's K outputs of this step
    if (x_.has_down && lane == kLatRows - 1 && (!(G || XL) || (tr - 31 >= 0 && tr - 31 < x_.Umax))) {
        float* dst = (!G && group_addr_ok<K>() && ga) ? ga->sdst + gs * K * 2 : x_.my_stream + size_t(tr - 31) * K * 2;
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
    // jf+16 (lanes 16-31), one coalesced 64-byte store per plane each.
    // Offsets are 32-bit, relative to the band's first output row.
    if (!G && group_addr_ok<K>() && ga) {
        bool ok = true;
        if (Y) {
            const int yf = y0 + ga->jf0 + gs - (K - 1);
            ok = yf >= 0 && yf < h;
        }
        if (XL) ok = ok && ga->seg_ok;
        if (ok) {
            const long long ro = (long long)gs * x_.opitch;
            const int o = ga->o0 + gs * OW;
            stg(ga->fo + ro, lds(o));
            stg(ga->bo + ro, lds(o + Gm::OPL));
        }
    } else {
        const int col = lane & (OW - 1);
        const int u = tr - (K - 1) - (OW - 1);
        const int jf = (u & (OW - 1)) + (lane & 16);
        const int xs = (u & ~(OW - 1)) - (lane & 16);  // segment start column (xf - 15)
        bool ok = true;
        if (G) {
            const int yf = y0 + jf - (K - 1);
            ok = xs >= 0 && xs + OW - 1 < w && yf >= 0 && yf < h;
        } else {
            if (Y) {
                const int yf = y0 + jf - (K - 1);
                ok = yf >= 0 && yf < h;
            }
            if (XL) ok = ok && xs >= 0;
        }
        if (ok) {  // off >= 0 here: unsigned, one IMAD.WIDE.U32 per plane
            const unsigned off = unsigned(jf * x_.opitch + xs + col);
            const int o = Gm::OFF_O + orow(jf) * OW + col;
            stg(x_.FO + off, lds(o));
            stg(x_.BO + off, lds(o + Gm::OPL));
        }
        if (G && ((w - 1) & (OW - 1)) != OW - 1) {  // partial last segment of a row
            const int je = tr - (K - 1) - (w - 1);
            const int x0 = (w - 1) & ~(OW - 1);
            const int ye = y0 + je - (K - 1);
            if (je >= 0 && je < 32 && ye >= 0 && ye < h && lane < w - x0) {
                const unsigned off = unsigned(je * x_.opitch + x0 + lane);
                const int o = Gm::OFF_O + orow(je) * OW + lane;
                stg(x_.FO + off, lds(o));
                stg(x_.BO + off, lds(o + Gm::OPL));
            }
        }
    }

    // every lane's flush reads are done before the next step's output-ring
    // stores reuse the slots (lanes of a diverged warp may run ahead)
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (G || Y || XL) st.rprev[k] = recv[k];
        st.outp[k] = nv[k];
    }
}

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

// Poll chunk `u0 / CK` of the band above until every word of it is
// written; leaves it in the chunk buffer.  `v` holds a load issued earlier
// and is re-polled only while incomplete.
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

// Poll chunk `u0 / CK` of the band above until every word of it is
// written; leaves it in the chunk buffer.  `v` holds a load issued earlier
// and is re-polled only while incomplete.  Bounded (SURVEY.md section 5,
// "timeout -> error, not a hang"): after spin_ns the wait raises the launch's
// abort flag, counts a device fault and returns false; every other waiter of
// the launch then gives up at once.
template <int K, int CK>
__device__ __forceinline__ bool acquire_chunk(float4 v, const float* up_stream, int u0, int Umax, int lane,
                                              int chunk, const SweepFail& F) {
    using G = Geom<K, CK>;
    const int nvalid = min(CK, Umax - u0) * K * 2;  // floats
    const bool mine = lane < G::CH4 && 4 * lane < nvalid;
    // (exponential back-off up to 4 us was measured: no effect on batches,
    // slower single images)
    // (the abort flag and the clock are checked every 256 polls only: a
    // check in every poll slows the hand-over of latency-bound launches)
    unsigned long long t0 = 0;
    for (unsigned n = 0; !__all_sync(kFull, chunk_complete<K, CK>(v, u0, Umax, lane)); ++n) {
        __nanosleep(32);
        if (mine) v = ld_relaxed_v4(up_stream + size_t(u0) * K * 2 + 4 * lane);
        if ((n & 255u) == 255u) {
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
    if (mine) sts4(chunk + 4 * lane, v);
    return true;
}


#ifndef FGM_REPOLL
#define FGM_REPOLL 1
#endif
template <int K, bool V4, int CK>
__device__ __forceinline__ void run_band(const SweepJob& J, int q, int ch, int lane, unsigned sbase, float eps,
                                         float omega, const SweepFail& F, int fault) {
    using Gm = Geom<K, CK>;
    const int w = J.w, h = J.h;
    const int y0 = q * kLatRows;
    const int Umax = w + K - 1;
    const size_t slen = sweep_stream_len(w, K);
    const int sid = q * 3 + ch;  // stream index of this (band, channel)
    const float* up_stream = q > 0 ? J.stream + size_t(sid - 3) * slen : nullptr;

    StepCtx<K> cx;
    cx.lb = lane * Gm::RS;
    cx.ob = Gm::OFF_O + orow(lane) * Gm::OW;
    cx.lane = lane;
    cx.y0 = y0;
    cx.w = w;
    cx.h = h;
    cx.has_up = q > 0;
    cx.has_down = q < J.nb - 1 && !(fault == 1 && q == 0);  // (fault 1: band 0 never publishes)
    cx.Umax = Umax;
    cx.my_stream = J.stream + size_t(sid) * slen;
    // band-relative output base (row y0 - (K-1) may be -1.. for the first
    // band: only the pointer arithmetic goes there, stores are bounds-checked)
    cx.FO = J.fg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    cx.BO = J.bg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    cx.opitch = J.opitch;
    cx.eps = eps;
    cx.omega = omega;

    // rows this lane streams
    const RowSrc own = make_rowsrc<K>(J, ch, y0, lane, true, true, true, sbase);
    const bool has_x = lane >= 32 - K || lane == 0;
    const RowSrc ext =
        make_rowsrc<K>(J, ch, y0, lane == 0 ? 32 : lane - 32, has_x, lane >= 33 - K, lane == 0, sbase);
#ifndef FGM_FLAT_ISSUE
#define FGM_FLAT_ISSUE 1
#endif
#if FGM_FLAT_ISSUE
    const FlatSrc<K> flat = make_flat<K, CK>(J, ch, y0, lane, sbase);
#endif

    LaneState<K> st;
#pragma unroll
    for (int k = 0; k < K; ++k) st.outp[k] = st.rprev[k] = make_float2(0.0f, 0.0f);

    // prologue: the loads "issued before" the first group, then M-1 empty
    // groups so that every group waits with the same cp.async.wait_group M-1
    constexpr int S = Gm::S;
    constexpr int t0 = -S;
    prologue_row<K, V4, CK>(own, t0, w);
    if (has_x) prologue_row<K, V4, CK>(ext, t0, w);
    cp_commit();
#pragma unroll
    for (int i = 1; i < Gm::M; ++i) cp_commit();
    // the band above's first chunk, polled when needed
    float4 pend = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool lane_ch = lane < Gm::CH4;
    bool pend_ok = false;  // pend holds the complete next chunk
    if (cx.has_up && lane_ch) pend = ld_relaxed_v4(up_stream + 4 * lane);

    // Border groups: bands touching row 0 or h-1, else the first and last ~32
    // steps.  Fast groups need no neighbour clamping and no bounds checks.
    const bool yband = y0 - (K - 1) <= 0 || y0 + 31 >= h - 1;
    const int fast_lo = 32 + K, fast_hi = w - 2;  // a step tr is fast iff fast_lo <= tr < fast_hi
    const int tend = 31 + Umax;                   // lane 31's last column is Umax-1
    // groups whose issued blocks are inside [0, w) for every row -K .. 32
    const int issue_lo = 32 - Gm::L, issue_hi = w - 2 * S - Gm::L - K;
    for (int t4 = t0; t4 < tend; t4 += S) {
        cp_wait<Gm::M - 1>();
        __syncwarp();
        if (t4 < 0) {
            // coefficients of step 0 (computed "at step -1")
            const int rc = cx.lb + ((-1 - lane - Gm::SH) & (Gm::RW - 1));
#pragma unroll
            for (int k = 0; k < K; ++k) st.co[k] = first_coef<K>(rc, k, -lane - k, y0 + lane - k, w, h, eps, omega);
        } else {
            if (cx.has_up && t4 < Umax) {
                const int nxt = (t4 & ~(CK - 1)) + CK;  // the next chunk's first column
                if ((t4 % CK) == 0) {
                    if (!acquire_chunk<K, CK>(pend, up_stream, t4, Umax, lane, Gm::OFF_C, F)) {
                        cp_wait<0>();  // the launch is aborted: drop the band
                        __syncwarp();
                        return;
                    }
                    pend_ok = false;
                    if (nxt < Umax && lane_ch)  // prefetch the next chunk
                        pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
                } else if (FGM_REPOLL && !pend_ok && nxt < Umax) {
                    // the prefetch found the next chunk incomplete: re-poll it
                    // now rather than a full round trip when it is needed
                    pend_ok = __all_sync(kFull, chunk_complete<K, CK>(pend, nxt, Umax, lane));
                    if (!pend_ok && lane_ch) pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
                }
            }
            __syncwarp();
            if (t4 >= fast_lo && t4 + S <= fast_hi && !yband) {
                const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll
                for (int s = 0; s < S; ++s) band_step<K, false, CK>(st, cx, t4 + s, &ga, s);
            } else if (t4 >= fast_lo && t4 + S <= fast_hi) {
                const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll
                for (int s = 0; s < S; ++s) band_step<K, false, CK, true>(st, cx, t4 + s, &ga, s);
            } else if (t4 < fast_lo && t4 + S <= fast_hi) {  // band start: left border only
                if (yband) {
                    const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll
                    for (int s = 0; s < S; ++s) band_step<K, false, CK, true, true>(st, cx, t4 + s, &ga, s);
                } else {
                    const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll
                    for (int s = 0; s < S; ++s) band_step<K, false, CK, false, true>(st, cx, t4 + s, &ga, s);
                }
            } else {
#pragma unroll 1
                for (int s = 0; s < S; ++s) band_step<K, true, CK>(st, cx, t4 + s);
            }
        }
        __syncwarp();  // every lane is done with the ring slots the next loads overwrite
        if (V4 && !yband && t4 >= issue_lo && t4 < issue_hi) {
#if FGM_FLAT_ISSUE
            issue_flat<K, CK>(flat, t4);
#else
            issue_row_fast<K, 15u, CK>(own, t4);
            issue_row_fast<K, 0u, CK>(ext, t4);
#endif
        } else {
            issue_row<K, V4, CK>(own, t4, w);
            if (has_x) issue_row<K, V4, CK>(ext, t4, w);
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

template <int K, bool V4, int CK>
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
        if (V4 && !J.vec4) {
            run_band<K, false, CK>(J, jb.y / 3, jb.y % 3, lane, sbase, A.eps, A.omega, A.fail, A.fault);
        } else {
            run_band<K, V4, CK>(J, jb.y / 3, jb.y % 3, lane, sbase, A.eps, A.omega, A.fail, A.fault);
        }
    }
}

// Per-device launch state: the function attributes (both chunk widths) and
// the resident-warp capacity.
template <int K>
cudaError_t sweep_grid_cap(int& cap) {
    static PerDevice<int> cfg;
    return cfg.get(cap, [](int dev, int& v) {
        const int sm4 = int(Geom<K, 4>::TOTAL * sizeof(float)), sm16 = int(Geom<K, kChunk>::TOTAL * sizeof(float));
        cudaError_t e = cudaFuncSetAttribute(sweep_kernel<K, true, kChunk>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm16);
        // the largest shared-memory carveout: the rings, not L1, bound the resident warps
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_kernel<K, true, kChunk>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_kernel<K, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_kernel<K, true, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int sms = 0, per_sm = 0;
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<K, true, kChunk>, 32, size_t(sm16));
        v = std::max(1, sms * std::max(1, per_sm));
        return e;
    });
}

// Launches whose (band, channel) items all fit on the GPU at once are
// latency-bound single images: their critical path crosses every band, one
// boundary-stream chunk per hand-over, so they poll 4-column chunks (a ~20%
// shorter hand-over lag); throughput launches poll 16-column chunks.
template <int K>
cudaError_t launch_sweep_k(const SweepArgs& A, cudaStream_t s) {
    int cap = 0;
    cudaError_t e = sweep_grid_cap<K>(cap);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(A.total, cap));
    if (A.total <= cap)
        sweep_kernel<K, true, 4><<<grid, 32, size_t(Geom<K, 4>::TOTAL) * sizeof(float), s>>>(A);
    else
        sweep_kernel<K, true, kChunk><<<grid, 32, size_t(Geom<K, kChunk>::TOTAL) * sizeof(float), s>>>(A);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_sweep_lat(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket,
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
