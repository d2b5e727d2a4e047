// K3, latency path: launches of a few images, whose time is the wavefront's
// dependency chain -- (w + h) steps of one lane plus the band hand-overs --
// not throughput.  Warp-specialised: one CTA per 32-row band, four warps.
//
//   warp 0, the producer: computes every pixel's alpha-only coefficients once
//     (edge weights, 1/S, alpha, 1/D: the rank-one solve of fgm_device.cuh,
//     multilevel.hpp:37-43 -- common to the three channels and to the K fused
//     sweeps) into a shared-memory ring, a few groups of steps ahead;
//   warps 1..3, the chains (colour channels 0..2): only the F_c/B_c
//     recurrence of their channel -- shuffle in the row above, the rank-one
//     update for K sweeps, output ring, boundary stream.
//
// Geometry as the throughput kernel with one row per lane: lane j owns skewed
// row j and at step t updates, for every sweep slot k < K, pixel
// (t - j - k, y0 + j - k).  Slot k of lane j needs the coefficients the
// producer made for row j - k at producer step t - 2k (pixel (x, y) of sweep k
// runs at step x + y + 2k); for lanes j < k that row is the band above's, whose
// producer publishes its last K-1 rows' coefficients in a per-band
// coefficient stream (sentinel-validated like the F/B streams).
//
// Producer and chains synchronise per group of 8 steps through mbarriers
// (full: producer -> chains; empty: chains -> producer, released one group
// late because slot k looks 2k steps back).  Each warp stages its own planes
// through 64-column shared-memory rings refilled in 16-column (64-byte) row
// segments (producer: alpha; chain c: I_c, initial F_c, B_c).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "fgm_device.cuh"
#include "fgm_internal.h"

namespace fgm {
namespace {

constexpr int BRW = kLatBandRows;  // band rows, one per lane
static_assert(BRW == 32, "one row per lane");
constexpr int GS = 8;              // steps per group (= boundary-stream chunk columns)
constexpr int NGR = 4;             // coefficient ring groups
constexpr int RL = GS * NGR;       // coefficient ring length (producer steps)

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
                 "f"(v.w));
}
__device__ __forceinline__ void st_relaxed_v2(float* p, float2 v) {
    asm volatile("st.relaxed.gpu.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y));
}
__device__ __forceinline__ bool is_sentinel(float v) { return __float_as_uint(v) == kStreamSentinel; }

extern __shared__ float4 ws_sm4[];
__device__ __forceinline__ float* wsf() { return reinterpret_cast<float*>(ws_sm4); }
__device__ __forceinline__ float lds(int i) { return wsf()[i]; }
__device__ __forceinline__ float2 lds2(int i) { return *reinterpret_cast<const float2*>(wsf() + i); }
__device__ __forceinline__ float4 lds4(int i) { return *reinterpret_cast<const float4*>(wsf() + i); }
__device__ __forceinline__ void sts2(int i, float2 v) { *reinterpret_cast<float2*>(wsf() + i) = v; }
__device__ __forceinline__ void sts4(int i, float4 v) { *reinterpret_cast<float4*>(wsf() + i) = v; }

// ---- mbarriers ---------------------------------------------------------------
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned a) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned a, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}

struct WsFail {
    int* abort_flag;
    int* fault_count;
    unsigned long long spin_ns;
};
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ bool launch_aborted(const WsFail& F) {
    return *reinterpret_cast<volatile int*>(F.abort_flag) != 0;
}

// Wait for an mbarrier phase; false if the launch was aborted meanwhile (a
// stalled hand-over elsewhere: every waiter gives up instead of hanging).
__device__ __forceinline__ bool mbar_wait(unsigned a, unsigned parity, const WsFail& F) {
    for (unsigned n = 0; !mbar_test(a, parity); ++n)
        if ((n & 63u) == 63u && launch_aborted(F)) return false;
    return true;
}

// ---- shared-memory geometry (floats) ----------------------------------------
//   producer: alpha ring, rows -1..32
//   coefficient ring: [RL steps][32 rows] x two float4 records:
//       A = (dL, dR, dU, dD), B = (1/S, alpha, 1/D, 0)
//   per chain warp: image ring rows -(K-1)..31, F and B rings rows 0..32,
//       output ring [orow 0..33][16 columns][F, B], F/B chunk [GS columns][K]
//       [F, B], coefficient chunk ring [2 GS columns][K-1][8]
//   mbarriers: full[NGR], empty[NGR]
// Rings are 64 columns (column x at x & 63), refilled in 16-column segments:
// a segment is issued 3 segments ahead of its slot's previous one leaving the
// read window, >= 34 steps before its first read (a lone chain steps in tens
// of nanoseconds: a shorter lead would expose DRAM latency).
template <int K>
struct WGeom {
    static constexpr int NA = BRW + 2, NI = BRW + K - 1, NF = BRW + 1;
    static constexpr int RW = 64;
    static constexpr int P_A = 0;
    static constexpr int NRR = BRW;  // ring rows per step slot
    static constexpr int RING = P_A + NA * RW;
    static constexpr int RING_B = RING + RL * NRR * 4;
    static constexpr int CH0 = RING_B + RL * NRR * 4;
    static constexpr int C_I = 0, C_F = C_I + NI * RW, C_B = C_F + NF * RW, C_O = C_B + NF * RW;
    static constexpr int OROWS = BRW + BRW / 16;
    static constexpr int C_CF = C_O + OROWS * 16 * 2;      // F/B chunk
    static constexpr int CHF = GS * K * 2;
    static constexpr int C_CC = C_CF + CHF;                // coefficient chunk ring: the band above's
    static constexpr int CCW = (K - 1) * 8;                // last K-1 rows, [2 GS columns][K-1][A, B]
    static constexpr int CHC = 2 * GS * CCW;
    static constexpr int CHAIN = (C_CC + CHC + 3) & ~3;
    static constexpr int BAR = CH0 + 3 * CHAIN;            // 2 * NGR uint64
    static constexpr int TOTAL = BAR + 4 * NGR;
};

__device__ __forceinline__ constexpr int orow(int r) { return r + (r >> 4); }

// Coefficient stream of a band: per column x, the K-1 records of its last K-1
// rows (rows 32-(K-1) .. 31), 8 floats each (sweep_cstream_len).
__device__ __forceinline__ size_t ws_cstream_len(int w, int K) { return sweep_cstream_len(w, K); }

// ---- ring refills -------------------------------------------------------------
constexpr int WRW = 64;  // ring columns

// One 16-byte piece (4 columns from c) of a plane row into a ring.
template <bool V4>
__device__ __forceinline__ void put_piece(const float* row, unsigned sdst_row, int c, int w, bool row_ok) {
    if (!row_ok || c < 0 || c >= w) return;
    const unsigned d = sdst_row + 4u * unsigned(c & (WRW - 1));
    const int nb = min(w - c, 4);
    if (V4) {
        cp_async16(d, row + c, nb * 4);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async4(d + 4 * i, i < nb ? row + c + i : row + c, i < nb ? 4 : 0);
    }
}

// A plane ring of rows lo .. lo+nrows-1 (band-relative), read window of row r
// at step t within [t - r + mlo, t - r + 1]: the segment n (16 columns) of row
// r is issued at step 16 (n-3) + r - mlo, when segment n-4 (same ring slot)
// has left the window; the group of steps [t0, t0 + GS) issues the rows whose
// issue step falls in it.  Lanes = (row within 8, piece); every piece
// checked (this path is latency-bound, not issue-bound).
template <bool V4>
__device__ __forceinline__ void refill_plane(const float* base, int pitch, unsigned sring, int lo, int nrows, int mlo,
                                             int t0, int lane, int y0, int w, int h) {
    const int q = lane & 3, rsub = lane >> 2;
    for (int r0 = 0; r0 < nrows; r0 += 8) {
        const int rr = r0 + rsub;
        if (rr >= nrows) break;
        const int r = lo + rr;
        // segments whose issue step 16 (n-3) + r - mlo lies in [t0, t0 + GS)
        const int z = t0 - r + mlo;  // 16 (n-3) in [z, z + GS)
        const int n3 = (z + 15) >> 4;  // ceil(z / 16) (arithmetic shift: floor division for negatives)
        const bool due = 16 * n3 < z + GS;
        const int c = 16 * (n3 + 3) + 4 * q;
        const int y = y0 + r;
        if (due && c >= WRW) put_piece<V4>(base + (long long)r * pitch, sring + 4u * unsigned(rr * WRW), c, w,
                                           y >= 0 && y < h);
    }
}

// Prologue: segments 0..3 (columns 0..63) of every ring row.
template <bool V4>
__device__ __forceinline__ void prologue_plane(const float* base, int pitch, unsigned sring, int lo, int nrows,
                                               int lane, int y0, int w, int h) {
    constexpr int PPR = WRW / 4;
    for (int it = lane; it < nrows * PPR; it += 32) {
        const int rr = it / PPR, r = lo + rr, y = y0 + r;
        put_piece<V4>(base + (long long)r * pitch, sring + 4u * unsigned(rr * WRW), 4 * (it % PPR), w,
                      y >= 0 && y < h);
    }
}

// ---- boundary-stream chunks -----------------------------------------------------
// The chunk of a group: GS columns of the band above's F/B stream (K pairs
// per column) followed by the same columns of its coefficient stream (K-1
// records of 8 floats), as float4 slots f = lane and lane + 32.  It is loaded
// one group ahead into registers and re-polled only while a word is still the
// sentinel (bounded).
template <int K>
struct ChunkPend {
    static constexpr int F4_FB = GS * K * 2 / 4, F4_CC = GS * (K - 1) * 8 / 4, F4 = F4_FB + F4_CC;
    static constexpr int NSLOT = (F4 + 31) / 32;
    static_assert(NSLOT <= 2, "chunk fits two float4 per lane");
    float4 v[NSLOT];
};

// valid floats of slot f for a chunk of ncol columns
template <int K>
__device__ __forceinline__ int chunk_valid(int f, int ncol) {
    using P = ChunkPend<K>;
    if (f < P::F4_FB) return min(4, ncol * K * 2 - 4 * f);
    if (f < P::F4) return min(4, ncol * (K - 1) * 8 - 4 * (f - P::F4_FB));
    return 0;
}
template <int K>
__device__ __forceinline__ const float* chunk_src(int f, const float* fb, const float* cc) {
    using P = ChunkPend<K>;
    return f < P::F4_FB ? fb + 4 * f : cc + 4 * (f - P::F4_FB);
}
template <int K>
__device__ __forceinline__ void chunk_issue(ChunkPend<K>& p, const float* fb, const float* cc, int ncol, int lane) {
    using P = ChunkPend<K>;
#pragma unroll
    for (int i = 0; i < P::NSLOT; ++i) {
        const int f = lane + 32 * i;
        if (chunk_valid<K>(f, ncol) > 0) p.v[i] = ld_relaxed_v4(chunk_src<K>(f, fb, cc));
    }
}
__device__ __forceinline__ bool words_ok(float4 v, int nvalid) {
    return !(is_sentinel(v.x) || (nvalid > 1 && is_sentinel(v.y)) || (nvalid > 2 && is_sentinel(v.z)) ||
             (nvalid > 3 && is_sentinel(v.w)));
}
// Complete the pending chunk (re-polling what is missing) and store it: F/B
// part at C_CF, coefficient part at C_CC + (t0 mod 2 GS) columns.
template <int K>
__device__ __forceinline__ bool chunk_acquire(ChunkPend<K>& p, const float* fb, const float* cc, int ncol, int lane,
                                              int chb, int t0, const WsFail& F) {
    using P = ChunkPend<K>;
    using G = WGeom<K>;
    unsigned long long tstart = 0;
    for (unsigned n = 0;; ++n) {
        bool mine = true;
#pragma unroll
        for (int i = 0; i < P::NSLOT; ++i) {
            const int f = lane + 32 * i, nv = chunk_valid<K>(f, ncol);
            if (nv > 0 && !words_ok(p.v[i], nv)) {
                mine = false;
            }
        }
        if (__all_sync(kFull, mine)) break;
        __nanosleep(32);
#pragma unroll
        for (int i = 0; i < P::NSLOT; ++i) {
            const int f = lane + 32 * i, nv = chunk_valid<K>(f, ncol);
            if (nv > 0 && !words_ok(p.v[i], nv)) p.v[i] = ld_relaxed_v4(chunk_src<K>(f, fb, cc));
        }
        if ((n & 255u) == 255u) {
            int ab = 0;
            if (lane == 0) {
                const unsigned long long now = global_ns();
                if (!tstart) tstart = now;
                ab = launch_aborted(F) ? 1 : 0;
                if (!ab && now - tstart > F.spin_ns) {
                    atomicExch(F.abort_flag, 1);
                    atomicAdd(F.fault_count, 1);
                    ab = 1;
                }
            }
            if (__shfl_sync(kFull, ab, 0)) return false;
        }
    }
#pragma unroll
    for (int i = 0; i < P::NSLOT; ++i) {
        const int f = lane + 32 * i;
        if (chunk_valid<K>(f, ncol) > 0) {
            const int d = f < P::F4_FB ? G::C_CF + 4 * f
                                       : G::C_CC + (t0 & (2 * GS - 1)) * G::CCW + 4 * (f - P::F4_FB);
            sts4(chb + d, p.v[i]);
        }
    }
    return true;
}

#ifdef FGM_WS_TRACE
__device__ unsigned long long g_ws_trace[8 * 4096];  // per band: start, chunk 0, step 64, step 512, end, producer start, producer step 64, 512
#endif

struct WsArgs {
    const SweepJob* jobs;
    const int2* order;  // (job, band * 3 + channel): every third entry is a band
    int total;          // bands
    unsigned* ticket;
    float eps, omega;
    WsFail fail;
    int fault;
};

// ---- the producer -------------------------------------------------------------
template <int K, bool V4>
__device__ __forceinline__ bool producer_band(const SweepJob& J, int q, int lane, unsigned sbase, float eps,
                                              float omega, const WsFail& F, unsigned& gseq, int ngroups) {
    using G = WGeom<K>;
    const int w = J.w, h = J.h, y0 = q * BRW;
    const float* abase = J.alpha + (long long)y0 * J.ipitch;
    const unsigned sA = sbase + 4u * unsigned(G::P_A);
    // the coefficient stream of this band (read by the band below)
    const bool pub = q < J.nb - 1;
    float* cstream = J.stream + size_t(J.nb) * 3 * sweep_stream_len(w, K) + size_t(q) * ws_cstream_len(w, K);
    const int prow = lane - (BRW - (K - 1));  // >= 0: this lane's row is published
#ifdef FGM_WS_TRACE
    if (lane == 0 && q < 4096) g_ws_trace[8 * q + 5] = global_ns();
#endif
    prologue_plane<V4>(abase, J.ipitch, sA, -1, G::NA, lane, y0, w, h);
#pragma unroll
    for (int i = 0; i < 4; ++i) cp_commit();  // (3 empty groups: the first wait_group 3 covers the prologue)
    const unsigned bar = sbase + 4u * unsigned(G::BAR);
    const int y = y0 + lane;
    const int row = G::P_A + (lane + 1) * G::RW;  // ring row of band row `lane` (rows from -1)
    const int rrow = lane;                        // coefficient-ring row
    const bool ytop = y <= 0, ybot = y >= h - 1;
    // (group -1: steps -8..-1 set up the carries of the first columns)
    for (int g = -1; g < ngroups; ++g, ++gseq) {
        const int t0 = g * GS;
        cp_wait<3>();
        __syncwarp();
        // the ring slots of this group are free once every chain has released
        // the group NGR back
        if (!mbar_wait(bar + 8u * (NGR + (gseq % NGR)), ((gseq / NGR) & 1u) ^ 1u, F)) return false;
#ifdef FGM_WS_TRACE
        if (lane == 0 && q < 4096 && t0 == 64) g_ws_trace[8 * q + 6] = global_ns();
        if (lane == 0 && q < 4096 && t0 == 512) g_ws_trace[8 * q + 7] = global_ns();
#endif
        const int xb = t0 - lane;  // x of step s = xb + s
        const bool xedge = xb - 1 <= 0 || xb + GS >= w - 1;
#pragma unroll
        for (int s = 0; s < GS; ++s) {
            const int x = xb + s;
            const float a = lds(row + (x & (G::RW - 1)));
            float aL = lds(row + ((x - 1) & (G::RW - 1))), aR = lds(row + ((x + 1) & (G::RW - 1)));
            float aU = lds(row - G::RW + (x & (G::RW - 1))), aD = lds(row + G::RW + (x & (G::RW - 1)));
            if (xedge) {
                if (x <= 0) aL = a;
                if (x >= w - 1) aR = a;
            }
            if (ytop) aU = a;
            if (ybot) aD = a;
            const float dL = edge_weight(a, aL, eps, omega), dR = edge_weight(a, aR, eps, omega);
            const float dU = edge_weight(a, aU, eps, omega), dD = edge_weight(a, aD, eps, omega);
            const float S = __fadd_rn(__fadd_rn(__fadd_rn(dL, dR), dU), dD);
            const f32x2 u = pk2(a, __fsub_rn(1.0f, a));
            const float2 uu = upk2(mul2(u, u));
            const float Dn = __fadd_rn(__fadd_rn(uu.x, uu.y), S);
            const float4 recA = make_float4(dL, dR, dU, dD);
            const float4 recB = make_float4(rcp_approx(S), a, rcp_approx(Dn), 0.0f);
            const int slot = ((t0 + s) & (RL - 1)) * G::NRR + rrow;
            sts4(G::RING + 4 * slot, recA);
            sts4(G::RING_B + 4 * slot, recB);
            if (pub && prow >= 0 && x >= 0 && x < w + K - 1) {
                // (columns past the row end: pixels outside the image, published
                // as zeros -- never the NaN sentinel of an unfilled ring slot)
                const bool in = x < w;
                float* dst = cstream + size_t(x) * G::CCW + prow * 8;
                st_relaxed_v4(dst, in ? recA : make_float4(0.f, 0.f, 0.f, 0.f));
                st_relaxed_v4(dst + 4, in ? recB : make_float4(0.f, 0.f, 0.f, 0.f));
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar + 8u * (gseq % NGR));  // full
        refill_plane<V4>(abase, J.ipitch, sA, -1, G::NA, -1, t0, lane, y0, w, h);
        cp_commit();
    }
    cp_wait<0>();
    __syncwarp();
    return true;
}

// ---- a chain warp ---------------------------------------------------------------
template <int K>
struct ChainState {
    float2 o[K];    // outputs of the previous step
    float2 rvp[K];  // the previous step's values from the row above (border self values)
    float2 FRp;     // the previous step's initial right neighbour (slot-0 self value)
};

struct ChainCtx {
    int lane, w, h, y0, Umax, opitch, chb;
    bool has_up, has_down;
    unsigned yflags;  // bit k: pixel row of slot k <= 0; bit 8 + k: >= h - 1 (constant over the band)
    float* my_stream;
    float* FO;
    float* BO;
};

// Step t = t0 + s.  B: some pixel of the step may be on or beyond an image
// border (x checks per step; row checks from the band's per-lane flags).
template <int K, bool B>
__device__ __forceinline__ void chain_step(ChainState<K>& st, const ChainCtx& c, int t0, int s) {
    using G = WGeom<K>;
    const int lane = c.lane, t = t0 + s, chb = c.chb;
    const int x0 = t - lane;
    // values from the row above: shfl.up of lane - 1, lane 0 from the F/B chunk
    float2 rv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) rv[k] = upk2(__shfl_up_sync(kFull, pk2(st.o[k]), 1));
    if (lane == 0 && c.has_up) {
#pragma unroll
        for (int k = 0; k < K; ++k) rv[k] = lds2(chb + G::C_CF + (t & (GS - 1)) * K * 2 + 2 * k);
    }
    const int cb = t0 - lane;  // x0 = cb + s; the index math below is common to the group's steps
    auto col = [&](int e) { return (cb + s + e) & (G::RW - 1); };
    const float2 FR = make_float2(lds(chb + G::C_F + lane * G::RW + col(1)), lds(chb + G::C_B + lane * G::RW + col(1)));
    const float2 FD =
        make_float2(lds(chb + G::C_F + (lane + 1) * G::RW + col(0)), lds(chb + G::C_B + (lane + 1) * G::RW + col(0)));
    float2 nv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        // coefficients of pixel (x0 - k, row lane - k): the ring's record of step
        // t - 2k, or (lanes < k) the band above's from the coefficient chunk
        int ia = G::RING + 4 * (((t0 + s - 2 * k) & (RL - 1)) * G::NRR + lane - k), ib = ia + (G::RING_B - G::RING);
        if (k > 0) {
            const int ic = chb + G::C_CC + ((((cb + s - k) & (2 * GS - 1)) * (K - 1)) + lane - k + K - 1) * 8;
            if (lane < k) {
                ia = ic;
                ib = ic + 4;
            }
        }
        const float4 A = lds4(ia);
        const float4 Bq = lds4(ib);
        const float I = lds(chb + G::C_I + (lane - k + K - 1) * G::RW + col(-k));
        CoefR co;
        co.dL = A.x;
        co.dR = A.y;
        co.dU = A.z;
        co.dD = A.w;
        co.iS = Bq.x;
        co.u = pk2(Bq.y, __fsub_rn(1.0f, Bq.y));
        co.pq = mul2(pk2(Bq.z, Bq.z), co.u);
        co.I = I;
        float2 L = st.o[k], U = rv[k];
        float2 R = k ? rv[k > 0 ? k - 1 : 0] : FR;
        float2 D = k ? st.o[k > 0 ? k - 1 : 0] : FD;
        if (B) {
            const float2 self = k ? st.rvp[k > 0 ? k - 1 : 0] : st.FRp;
            const int x = x0 - k;
            if (x <= 0) L = self;
            if (x >= c.w - 1) R = self;
            if ((c.yflags >> k) & 1u) U = self;
            if ((c.yflags >> (8 + k)) & 1u) D = self;
        }
        nv[k] = pixel_applyr(co, L, R, U, D);
    }
    // output ring (last slot), column x & 15, (F, B) interleaved
    sts2(chb + G::C_O + (orow(lane) * 16 + ((cb + s - (K - 1)) & 15)) * 2, nv[K - 1]);
    // boundary stream for the band below
    if (c.has_down && lane == BRW - 1) {
        const int u = t - (BRW - 1);
        if (!B || (u >= 0 && u < c.Umax)) {
            float* dst = c.my_stream + size_t(u) * K * 2;
            if (K % 2 == 0) {
#pragma unroll
                for (int k = 0; k + 1 < K; k += 2)
                    st_relaxed_v4(dst + 2 * k, make_float4(nv[k].x, nv[k].y, nv[k + 1].x, nv[k + 1].y));
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) st_relaxed_v2(dst + 2 * k, nv[k]);
            }
        }
    }
    __syncwarp();
    // flush the 16-column segments completed at this step: rows rho (lanes
    // 0-15) and rho + 16 (lanes 16-31)
    {
        const int rho = (t - K - 14) & 15;
        const int r = rho + (lane & 16), cl = lane & 15;
        const int xs = t - K + 1 - r - 15;
        const int x = xs + cl;
        bool ok = true;
        if (B) ok = xs >= 0 && x < c.w && unsigned(c.y0 + r - (K - 1)) < unsigned(c.h);
        if (ok) {
            const float2 v = lds2(chb + G::C_O + (orow(r) * 16 + cl) * 2);
            const long long off = (long long)r * c.opitch + x;
            __stcg(c.FO + off, v.x);
            __stcg(c.BO + off, v.y);
        }
        if (B && ((c.w - 1) & 15) != 15) {  // the partial last segment of a row
            const int re = t - (K - 1) - (c.w - 1);
            const int xb = (c.w - 1) & ~15;
            const int ye = c.y0 + re - (K - 1);
            if (re >= 0 && re < BRW && ye >= 0 && ye < c.h && lane < c.w - xb) {
                const float2 v = lds2(chb + G::C_O + (orow(re) * 16 + lane) * 2);
                const long long off = (long long)re * c.opitch + xb + lane;
                __stcg(c.FO + off, v.x);
                __stcg(c.BO + off, v.y);
            }
        }
    }
    // every lane's flush reads are done before the next step's output-ring
    // stores reuse the slots (lanes of a diverged warp may run ahead)
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        st.rvp[k] = rv[k];
        st.o[k] = nv[k];
    }
    st.FRp = FR;
}

template <int K, bool V4>
__device__ __forceinline__ bool chain_band(const SweepJob& J, int q, int ch, int lane, unsigned sbase, float eps,
                                           const WsFail& F, int fault, unsigned& gseq, int ngroups) {
    using G = WGeom<K>;
    (void)eps;
    const int w = J.w, h = J.h, y0 = q * BRW;
    const int Umax = w + K - 1;
    const size_t slen = sweep_stream_len(w, K);
    const int sid = q * 3 + ch;
    const bool has_up = q > 0, has_down = q < J.nb - 1 && !(fault == 1 && q == 0);
    const float* up_stream = has_up ? J.stream + size_t(sid - 3) * slen : nullptr;
    // (K = 1 has no coefficient stream: its chunk part is empty)
    const float* up_cstream =
        has_up ? J.stream + size_t(J.nb) * 3 * slen + size_t(q - 1) * ws_cstream_len(w, K) : J.stream;
    float* my_stream = J.stream + size_t(sid) * slen;
    float* FO = J.fg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    float* BO = J.bg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    const int chb = G::CH0 + ch * G::CHAIN;
    const unsigned sch = sbase + 4u * unsigned(chb);
    const float* ibase = J.img + (long long)ch * J.istride + (long long)y0 * J.ipitch;
    const float* fbase = J.fg_in + (long long)ch * J.fstride + (long long)y0 * J.fpitch;
    const float* bbase = J.bg_in + (long long)ch * J.fstride + (long long)y0 * J.fpitch;
    constexpr int MI = -2 * (K - 1);
    prologue_plane<V4>(ibase, J.ipitch, sch + 4u * G::C_I, -(K - 1), G::NI, lane, y0, w, h);
    prologue_plane<V4>(fbase, J.fpitch, sch + 4u * G::C_F, 0, G::NF, lane, y0, w, h);
    prologue_plane<V4>(bbase, J.fpitch, sch + 4u * G::C_B, 0, G::NF, lane, y0, w, h);
#pragma unroll
    for (int i = 0; i < 4; ++i) cp_commit();
    // band 0: no band above -- zero chunks (finite values for the pixels above the image)
    for (int i = lane; i < G::CHF + G::CHC; i += 32) wsf()[chb + G::C_CF + i] = 0.0f;
    ChainState<K> st;
#pragma unroll
    for (int k = 0; k < K; ++k) st.o[k] = st.rvp[k] = make_float2(0.0f, 0.0f);
    st.FRp = make_float2(0.0f, 0.0f);
    const unsigned bar = sbase + 4u * unsigned(G::BAR);
    ChunkPend<K> pend;
#pragma unroll
    for (int i = 0; i < ChunkPend<K>::NSLOT; ++i) pend.v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (has_up) chunk_issue<K>(pend, up_stream, up_cstream, min(GS, Umax), lane);
    ChainCtx cx;
    cx.lane = lane;
    cx.w = w;
    cx.h = h;
    cx.y0 = y0;
    cx.Umax = Umax;
    cx.opitch = J.opitch;
    cx.chb = chb;
    cx.has_up = has_up;
    cx.has_down = has_down;
    cx.my_stream = my_stream;
    cx.FO = FO;
    cx.BO = BO;
    cx.yflags = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int yk = y0 + lane - k;
        if (yk <= 0) cx.yflags |= 1u << k;
        if (yk >= h - 1) cx.yflags |= 1u << (8 + k);
    }
    // steps t0..t0+GS-1 are interior iff every pixel has 1 <= x <= w - 2, every
    // flushed segment starts at x >= 0 and the stream slot is in range, and no
    // row of the band is at the top or bottom
    const bool yband = y0 - (K - 1) <= 0 || y0 + BRW - 1 >= h - 1;
    const int fast_lo = 31 + 15 + K, fast_hi = w - 2;
    bool ok = true;
#ifdef FGM_WS_TRACE
    const bool trace = ch == 0 && lane == 0 && q < 4096;
    if (trace) g_ws_trace[8 * q] = global_ns();
#endif
    // (group -1: steps -8..-1 set up the carries of the first columns)
    for (int g = -1; g < ngroups; ++g, ++gseq) {
        const int t0 = g * GS;
#ifdef FGM_WS_TRACE
        if (trace && t0 == 64) g_ws_trace[8 * q + 2] = global_ns();
        if (trace && t0 == 512) g_ws_trace[8 * q + 3] = global_ns();
#endif
        cp_wait<3>();
        __syncwarp();
        if (has_up && t0 >= 0 && t0 < Umax) {
            if (!chunk_acquire<K>(pend, up_stream + size_t(t0) * K * 2, up_cstream + size_t(t0) * G::CCW,
                                  min(GS, Umax - t0), lane, chb, t0, F)) {
                ok = false;
                break;
            }
#ifdef FGM_WS_TRACE
            if (trace && t0 == 0) g_ws_trace[8 * q + 1] = global_ns();
#endif
            const int tn = t0 + GS;  // prefetch the next group's chunk
            if (tn < Umax)
                chunk_issue<K>(pend, up_stream + size_t(tn) * K * 2, up_cstream + size_t(tn) * G::CCW,
                               min(GS, Umax - tn), lane);
        }
        if (!mbar_wait(bar + 8u * (gseq % NGR), (gseq / NGR) & 1u, F)) {  // this group's coefficients
            ok = false;
            break;
        }
        __syncwarp();
        if (!yband && t0 >= fast_lo && t0 + GS - 1 <= fast_hi) {
#pragma unroll
            for (int s = 0; s < GS; ++s) chain_step<K, false>(st, cx, t0, s);
        } else {
#pragma unroll
            for (int s = 0; s < GS; ++s) chain_step<K, true>(st, cx, t0, s);
        }
        __syncwarp();
        // release the group before (slot k looks 2k < GS steps back)
        if (g > -1 && lane == 0) mbar_arrive(bar + 8u * (NGR + ((gseq - 1) % NGR)));
        refill_plane<V4>(ibase, J.ipitch, sch + 4u * G::C_I, -(K - 1), G::NI, MI, t0, lane, y0, w, h);
        refill_plane<V4>(fbase, J.fpitch, sch + 4u * G::C_F, 0, G::NF, 1, t0, lane, y0, w, h);
        refill_plane<V4>(bbase, J.fpitch, sch + 4u * G::C_B, 0, G::NF, 1, t0, lane, y0, w, h);
        cp_commit();
    }
    if (ok && lane == 0) mbar_arrive(bar + 8u * (NGR + ((gseq - 1) % NGR)));  // the last group
#ifdef FGM_WS_TRACE
    if (trace) g_ws_trace[8 * q + 4] = global_ns();
#endif
    cp_wait<0>();
    __syncwarp();
    return ok;
}

template <int K>
__global__ void __launch_bounds__(128, 1) sweep_ws_kernel(WsArgs A) {
    using G = WGeom<K>;
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(ws_sm4));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    __shared__ unsigned s_ticket;
    const unsigned bar = sbase + 4u * unsigned(G::BAR);
    if (tid < 2 * NGR) mbar_init(bar + 8u * tid, tid < NGR ? 1u : 3u);  // full: producer; empty: 3 chains
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned gseq = 0;  // groups processed so far (every warp counts the same)
    for (;;) {
        if (tid == 0) s_ticket = atomicAdd(A.ticket, 1u);
        __syncthreads();
        const unsigned tk = s_ticket;
        if (tk >= unsigned(A.total) || launch_aborted(A.fail)) return;
        const int2 jb = A.order[3 * tk];
        const SweepJob J = A.jobs[jb.x];
        const int q = jb.y / 3;
        const int ngroups = (J.w + K - 1 + BRW - 1 + GS - 1) / GS;
        bool ok;
        if (warp == 0)
            ok = J.vec4 ? producer_band<K, true>(J, q, lane, sbase, A.eps, A.omega, A.fail, gseq, ngroups)
                        : producer_band<K, false>(J, q, lane, sbase, A.eps, A.omega, A.fail, gseq, ngroups);
        else
            ok = J.vec4 ? chain_band<K, true>(J, q, warp - 1, lane, sbase, A.eps, A.fail, A.fault, gseq, ngroups)
                        : chain_band<K, false>(J, q, warp - 1, lane, sbase, A.eps, A.fail, A.fault, gseq, ngroups);
        (void)ok;
        __syncthreads();
        if (launch_aborted(A.fail)) return;
    }
}

template <int K>
cudaError_t ws_grid_cap(int& cap) {
    static PerDevice<int> cfg;
    return cfg.get(cap, [](int dev, int& v) {
        const int sm = int(WGeom<K>::TOTAL * sizeof(float));
        cudaError_t e = cudaFuncSetAttribute(sweep_ws_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_ws_kernel<K>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int sms = 0, per_sm = 0;
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_ws_kernel<K>, 128, size_t(sm));
        v = std::max(1, sms * std::max(1, per_sm));
        return e;
    });
}

template <int K>
cudaError_t launch_ws_k(const WsArgs& A, cudaStream_t s) {
    int cap = 0;
    cudaError_t e = ws_grid_cap<K>(cap);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(A.total, cap));
    sweep_ws_kernel<K><<<grid, 128, size_t(WGeom<K>::TOTAL) * sizeof(float), s>>>(A);
    return cudaGetLastError();
}

}  // namespace

#ifdef FGM_WS_TRACE
extern "C" int fgm_debug_ws_trace(unsigned long long* out, int n) {
    return int(cudaMemcpyFromSymbol(out, g_ws_trace, size_t(n) * sizeof(unsigned long long)));
}
#endif

cudaError_t launch_sweep_ws(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_items,
                            unsigned* ticket, float eps, float omega, int* abort_flag, int* fault_count,
                            cudaStream_t s) {
    WsArgs A;
    A.jobs = jobs_dev;
    A.order = order_dev;
    A.total = total_items / 3;  // bands
    A.ticket = ticket;
    A.eps = eps;
    A.omega = omega;
    A.fail.abort_flag = abort_flag;
    A.fail.fault_count = fault_count;
    A.fail.spin_ns = (unsigned long long)std::max<long long>(g_spin_timeout_ns.load(), 1000);
    A.fault = g_sweep_fault.load();
    switch (K) {
        case 1: return launch_ws_k<1>(A, s);
        case 2: return launch_ws_k<2>(A, s);
        case 3: return launch_ws_k<3>(A, s);
        case 4: return launch_ws_k<4>(A, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fgm
