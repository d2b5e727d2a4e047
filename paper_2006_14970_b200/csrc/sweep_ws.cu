// K3, latency path: the warp-specialised sweep kernel for launches of a few
// images, whose time is the wavefront's dependency chain ((w + h) steps of one
// lane, plus ~36 steps per band hand-over), not throughput.  One CTA of eight
// warps per 32-row band:
//
//   * two producer warps compute every pixel's alpha-only coefficients (the
//     2x2 matrix is shared by all channels, multilevel.hpp:37-43) ONCE, ahead
//     of the wavefront, into a shared-memory record ring
//     {dL, dD, dR, dU | 1/S, a, u0/D, u1/D} (alternate groups of four steps
//     each, from their own alpha rings);
//   * three chain warps (one per colour channel) run only the recurrence of
//     multilevel.cpp:104-118: receive the previous lane's outputs (shfl), load
//     the records of their K pixels (two LDS.128 each), apply (pixel_applyr),
//     store into a 32-column output ring.  A group of four steps is
//     straight-line code with no barrier, no cp.async and no global store
//     except lane 31's boundary-stream words;
//   * three helper warps (one per channel) stream the channel's I_c and initial
//     F_c / B_c rows into shared-memory rings ahead of the chain warp (cp.async)
//     and flush its completed 16-column output segments behind it.
//
// Neither the producers nor the helpers depend on the band above, so a band's
// coefficients and ring data are in shared memory long before its first
// boundary chunk arrives: a band start, which is on the chain's critical
// path, waits for nothing but the chunk.
//
// The warps synchronise through monotonic progress counters in shared memory
// (volatile, cached by the reader; see st_volatile_cta): a chain warp starts
// group n once its helper has published the group's ring data and the
// producers have finished groups n and n + 1; a producer starts group P once
// every chain warp works on group >= P - 4 (record slots are reused after 32
// columns = 8 groups); a helper runs iteration i (flush group i - 1, issue the
// blocks that overwrite columns last read in group i - 1) once its chain warp
// has finished group i - 1.  Every wait is bounded (the launch's abort flag
// and spin timeout).
//
// Geometry, boundary streams, ticket order and border handling are those of
// lane j of a chain warp owns skewed row v = 32q + j and
// at step t updates, for every k < K, pixel (t - j - k, y0 + j - k); lane 0
// reads the band above's last lane from its boundary stream (NaN-sentinel
// words, no fences), lane 31 publishes this band's.  The arithmetic is
// pixel_coefr_dl / pixel_applyr of fgm_device.cuh, operation for operation:
// results are bitwise those of the throughput kernel (sweep.cu).
//
// -DFGM_WS_TRACE: per-phase cycle counts and a band timeline (printf) for
// development; profiles/r02/k3_ws_notes.txt.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>

#include "fgm_device.cuh"
#include "fgm_internal.h"

namespace fgm {
namespace {

constexpr int kRows = kLatBandRows;  // band rows (one per lane)
constexpr int kAhead = 4;            // producer group P needs every chain warp on group >= P - kAhead

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
// (no "memory" clobber: every stream word validates itself, so the stores
// need no ordering against this warp's other memory operations)
__device__ __forceinline__ void st_relaxed_v4(float* p, float4 v) {
    asm volatile("st.relaxed.gpu.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
}
__device__ __forceinline__ void st_relaxed_v2(float* p, float2 v) {
    asm volatile("st.relaxed.gpu.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y));
}
// The progress protocol runs without fences (a fence drains the warp's
// outstanding cp.async and global stores: 200-700 cycles per group, measured
// with st.release / ld.acquire): shared-memory accesses of one SM are served
// in issue order, so a volatile store issued after the warp's record accesses
// (__syncwarp) cannot overtake them, and record reads issued after a volatile
// load that saw the counter see the records stored before it.
__device__ __forceinline__ void st_volatile_cta(unsigned saddr, int v) {
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_cta(unsigned saddr) {
    int v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
    return v;
}

extern __shared__ float4 ws_sm4[];
__device__ __forceinline__ float* smf() { return reinterpret_cast<float*>(ws_sm4); }
__device__ __forceinline__ float lds(int i) { return smf()[i]; }
__device__ __forceinline__ float4 lds4(int i) { return reinterpret_cast<const float4*>(smf() + i)[0]; }
__device__ __forceinline__ void sts(int i, float v) { smf()[i] = v; }
__device__ __forceinline__ void sts4(int i, float4 v) { reinterpret_cast<float4*>(smf() + i)[0] = v; }
__device__ __forceinline__ void stg(float* p, float v) { __stcg(p, v); }
__device__ __forceinline__ bool is_sentinel(float v) { return __float_as_uint(v) == kStreamSentinel; }

// Shared-memory layout of one band CTA, in floats.
//
// Chain warps (per channel): rings of 32 columns per row for I_c (band rows
// -(K-1)..31) and the initial F_c, B_c (rows 0..32), column x at x mod 32 with
// the first MIR columns mirrored after column 31, so every read of a step is
// lane_base + c + (compile-time offset) with one c = (t - lane - SH) mod 32.
// Rows are RS = 32 + MIR floats apart (RS - 1 odd: the diagonal reads of a
// step hit distinct banks).  Loads run in groups of S = 4 steps with a lead of
// L columns, M groups in flight.  The output ring has 32 columns per row:
// 16-column segments are flushed once per group.
// Records: two float4 arrays [row -(K-1)..31][32 + MIR] with the same ring.
// Producer: an alpha ring of 64 columns for rows -K..32, MA groups in flight.
template <int K, int CK = kChunk>
struct Geom {
    static constexpr int RW = 32;
    static constexpr int SH = K - 1;
    static constexpr int MIR = K <= 2 ? 4 : 8;
    static constexpr int RS = RW + MIR;
    static constexpr int S = 4;
    static constexpr int M = 4;
    static constexpr int L = S * M + 1;
    static constexpr int NI = 31 + K;
    static constexpr int NF = 33;
    static constexpr int OW = 32;   // output ring columns
    static constexpr int SEG = 16;  // flushed segment
    // per-channel region
    static constexpr int C_I = 0;
    static constexpr int C_F = C_I + NI * RS;
    static constexpr int C_B = C_F + NF * RS;
    static constexpr int C_O = C_B + NF * RS;  // [plane F/B][row][OW]
    static constexpr int OPL = kRows * OW;
    static constexpr int C_C = C_O + 2 * OPL;
    static constexpr int CH = CK * K * 2;  // one boundary-stream chunk [u][k][F,B]
    static constexpr int CH4 = CH / 4;
    static constexpr int CHSZ = (C_C + kChunk * K * 2 + 3) / 4 * 4;  // (the same layout for every CK)
    // CTA-wide regions
    static constexpr int NR = 31 + K;  // record rows: band rows -(K-1)..31
    static constexpr int REC_A = 3 * CHSZ;
    static constexpr int REC_B = REC_A + NR * RS * 4;
    static constexpr int AW = 64;        // alpha ring columns
    static constexpr int ARS = AW + 4;   // ARS - 1 odd
    static constexpr int NA = 33 + K;    // alpha ring rows: band rows -K..32
    static constexpr int MA = 4;         // alpha load iterations in flight (an iteration: 2S columns)
    static constexpr int LA = 2 * S * MA;  // alpha load lead: 2S*MA - S + 3 + W1, W1 = 1
    static constexpr int OFF_AL = REC_B + NR * RS * 4;
    static constexpr int OFF_PR = OFF_AL + 2 * NA * ARS;  // progress words (one alpha ring per producer)
    static constexpr int PR_PROD = 0;                     // producers 0, 1: iterations finished
    static constexpr int PR_CHAIN = 2;                    // chain warps 0..2: groups finished
    static constexpr int PR_LOAD = 5;                     // helpers 0..2: chain groups whose ring data has landed
    static constexpr int NPR = 8;
    static constexpr int TOTAL = OFF_PR + NPR;
    static_assert(L + 3 + (2 * K - 3) + 2 * S <= RW + 3, "image ring too small for its lead");
    static_assert(K + 1 <= MIR && MIR % 4 == 0 && RS % 4 == 0, "mirror too narrow");
    static_assert(CH % 4 == 0 && CH4 <= 32, "a chunk is at most one float4 per lane");
    static_assert(LA + S + 3 + 2 <= AW, "alpha ring too small for its lead");
    static_assert(CHSZ % 4 == 0 && REC_A % 4 == 0 && OFF_AL % 4 == 0, "16-byte alignment");
};

// ---- chain warps: I_c / F_c / B_c ring loads --------------------------------

// The global rows a lane streams into its rings: its own band row and, for
// some lanes, one extra row (image rows -(K-1)..-1, F/B row 32).
struct RowSrc {
    const float* g[3];  // image c, F_c, B_c rows (column 0)
    unsigned s;         // shared address of channel offset 0, ring row r, column 0
    unsigned vm;        // bit p: plane p is streamed
    int r;              // row relative to the band
};

template <int K>
__device__ __forceinline__ constexpr int plane_off(int p) {
    using G = Geom<K>;
    return p == 0 ? G::C_I + (K - 1) * G::RS : p == 1 ? G::C_F : G::C_B;
}

template <int K>
__device__ __forceinline__ RowSrc make_rowsrc(const SweepJob& J, int ch, int y0, int r, bool doI, bool doF,
                                              unsigned cbase) {
    using G = Geom<K>;
    RowSrc rs;
    const int y = y0 + r;
    const bool ok = y >= 0 && y < J.h;
    const long long oi = (long long)(ok ? y : 0) * J.ipitch, of = (long long)(ok ? y : 0) * J.fpitch;
    rs.g[0] = J.img + ch * J.istride + oi;
    rs.g[1] = J.fg_in + ch * J.fstride + of;
    rs.g[2] = J.bg_in + ch * J.fstride + of;
    rs.s = cbase + 4u * unsigned(r * G::RS);  // may wrap below cbase: only ever offset back into range
    rs.vm = ok ? (doI ? 1u : 0u) | (doF ? 6u : 0u) : 0u;
    rs.r = r;
    return rs;
}

// cp.async of the S-column block at column x0 of every streamed plane of one
// row (general path: range checks, zero-fill past the row end).
template <int K, bool V4>
__device__ __forceinline__ void put_blocks(const RowSrc& rs, int x0, int w) {
    using G = Geom<K>;
    if (x0 < 0 || x0 >= w) return;
    const int nb = min(w - x0, 4) * 4;
    const int c = x0 & (G::RW - 1);
    const unsigned sc = rs.s + 4u * c;
    const bool mir = c < G::MIR;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        if (!(rs.vm & (1u << p))) continue;
        const float* g = rs.g[p] + x0;
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

template <int K, bool V4>
__device__ __forceinline__ void issue_row(const RowSrc& rs, int t4, int w) {
    using G = Geom<K>;
    put_blocks<K, V4>(rs, (t4 + G::S + G::L - rs.r) & ~(G::S - 1), w);
}

template <int K, bool V4>
__device__ __forceinline__ void prologue_row(const RowSrc& rs, int t0, int w) {
    using G = Geom<K>;
    const int last = (t0 + G::L - rs.r) & ~(G::S - 1);  // the block issued at the end of group t0 - S
    for (int x0 = 0; x0 <= last; x0 += G::S) put_blocks<K, V4>(rs, x0, w);
}

// Interior groups of interior bands, flattened: the 97 + K (plane, band row)
// blocks a group issues are dealt to the lanes of 4 cp.async instructions.
template <int K>
struct FlatSrc {
    static constexpr int N = (97 + K + 31) / 32;
    const float* g[N];
    unsigned s[N];
    int q[N];
    unsigned on;
};

template <int K>
__device__ __forceinline__ FlatSrc<K> make_flat(const SweepJob& J, int ch, int y0, int lane, unsigned cbase) {
    using G = Geom<K>;
    FlatSrc<K> f;
    f.on = 0;
    constexpr int NIm = 31 + K, NFB = 33;
#pragma unroll
    for (int i = 0; i < FlatSrc<K>::N; ++i) {
        int it = 32 * i + lane;
        int p = 0, r = 0;
        if (it < NIm) {
            p = 0;
            r = it - (K - 1);
        } else if ((it -= NIm) < NFB) {
            p = 1;
            r = it;
        } else if ((it -= NFB) < NFB) {
            p = 2;
            r = it;
        } else {
            p = -1;
        }
        const int y = min(max(y0 + r, 0), J.h - 1);  // (clamped for the first and last band: such ring rows are never read)
        const float* base = p == 0 ? J.img + ch * J.istride + (long long)y * J.ipitch
                          : p == 1 ? J.fg_in + ch * J.fstride + (long long)y * J.fpitch
                                   : J.bg_in + ch * J.fstride + (long long)y * J.fpitch;
        f.g[i] = base;
        const int po = p == 0 ? plane_off<K>(0) : p == 1 ? plane_off<K>(1) : plane_off<K>(2);
        f.s[i] = cbase + 4u * unsigned(po + r * G::RS);
        f.q[i] = G::S + G::L - r;
        if (p >= 0) f.on |= 1u << i;
    }
    return f;
}

// LO: a band's first groups, where the blocks of the lower rows are still left
// of column 0 (skipped).
template <int K, bool LO = false>
__device__ __forceinline__ void issue_flat(const FlatSrc<K>& f, int t4) {
    using G = Geom<K>;
#pragma unroll
    for (int i = 0; i < FlatSrc<K>::N; ++i) {
        const int xs = (t4 + f.q[i]) & ~(G::S - 1);
        const unsigned x0 = unsigned(LO ? max(xs, 0) : xs);
        const unsigned c = x0 & (G::RW - 1);
        const float* g = f.g[i] + x0;
        const unsigned d = f.s[i] + 4u * c;
        const unsigned on = (f.on >> i) & (LO ? (xs >= 0 ? 1u : 0u) : 1u);
        cp_async16_if(d, g, on);
        cp_async16_if(d + 4u * G::RW, g, on & (c < unsigned(G::MIR) ? 1u : 0u));
    }
}

// ---- launch-wide failure state and bounded waits ----------------------------

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

// One bounded-wait check, every 256 polls of a spin: false = give up (the
// launch is aborted, or this wait exceeded spin_ns and aborts it).
// (The slow paths of the waits are out of line: the chain warp's per-group
// control code stays small and next to its step block in the instruction
// cache; ncu shows stall_no_instruction leading in the inlined wait code.)
// (everything by value: a reference would put the caller's variable on the stack)
__device__ __noinline__ unsigned long long keep_waiting_check(unsigned long long t0, int lane, SweepFail F) {
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
    t0 = __shfl_sync(kFull, t0, 0);
    return __shfl_sync(kFull, ab, 0) ? ~0ull : t0;  // ~0: give up
}
__device__ __forceinline__ bool keep_waiting(unsigned n, unsigned long long& t0, int lane, const SweepFail& F) {
    if ((n & 255u) != 255u) return true;
    t0 = keep_waiting_check(t0, lane, F);
    return t0 != ~0ull;
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

// Poll chunk u0 / CK of the band above until every word of it is written;
// leaves it in the chunk buffer.  `v` holds a load issued earlier and is
// re-polled only while incomplete.
struct ChunkPoll {
    float4 v;
    bool ok;
};
template <int K, int CK>
__device__ __noinline__ ChunkPoll acquire_chunk_spin(const float* up_stream, int u0, int Umax, int lane, SweepFail F) {
    using G = Geom<K, CK>;
    const int nvalid = min(CK, Umax - u0) * K * 2;
    const bool mine = lane < G::CH4 && 4 * lane < nvalid;
    unsigned long long t0 = 0;
    ChunkPoll r;
    r.v = make_float4(0.f, 0.f, 0.f, 0.f);
    r.ok = true;
    for (unsigned n = 0;; ++n) {
        if (CK > 4) __nanosleep(32);  // (4-column chunks: latency-bound launches, the load's round trip is the poll interval)
        if (mine) r.v = ld_relaxed_v4(up_stream + size_t(u0) * K * 2 + 4 * lane);
        if (__all_sync(kFull, chunk_complete<K, CK>(r.v, u0, Umax, lane))) return r;
        if (!keep_waiting(n, t0, lane, F)) {
            r.ok = false;
            return r;
        }
    }
}
template <int K, int CK>
__device__ __forceinline__ bool acquire_chunk(float4 v, const float* up_stream, int u0, int Umax, int lane,
                                              int chunk, const SweepFail& F) {
    using G = Geom<K, CK>;
    if (!__all_sync(kFull, chunk_complete<K, CK>(v, u0, Umax, lane))) {
        const ChunkPoll r = acquire_chunk_spin<K, CK>(up_stream, u0, Umax, lane, F);
        if (!r.ok) return false;
        v = r.v;
    }
    const int nvalid = min(CK, Umax - u0) * K * 2;
    if (lane < G::CH4 && 4 * lane < nvalid) sts4(chunk + 4 * lane, v);
    return true;
}

// Wait until the progress word at `saddr` reaches `need` (a monotonic
// counter); returns the value seen, or -1 when aborted.  Called by a converged
// warp: every lane reads the same word in the same instruction (a broadcast),
// so the value and the branches on it are warp-uniform.
__device__ __noinline__ int wait_progress_spin(unsigned saddr, int need, int lane, SweepFail F) {
    unsigned long long t0 = 0;
    for (unsigned n = 0;; ++n) {
        if (!keep_waiting(n, t0, lane, F)) return -1;
        const int v = ld_volatile_cta(saddr);
        if (v >= need) return v;
    }
}
__device__ __forceinline__ int wait_progress(unsigned saddr, int need, int lane, const SweepFail& F) {
    const int v = ld_volatile_cta(saddr);
    return v >= need ? v : wait_progress_spin(saddr, need, lane, F);
}

// ---- chain warps -------------------------------------------------------------

template <int K>
struct LaneState {
    float2 outp[K];   // this lane's (F_c, B_c) outputs of the previous step
    float2 rprev[K];  // what this lane received from lane-1 at the previous step (border steps)
    CoefR co[K];      // this step's coefficients (loaded one step ahead)
};

template <int K>
struct ChainCtx {
    int cb;   // float index of the channel region
    int lb;   // cb + lane * RS: ring offset 0, row "lane", column 0
    int rb;   // 4 * lane * RS: record float index of row "lane", column 0 (relative to REC_A / REC_B)
    int lane, y0, w, h;
    bool has_up, has_down;
    int Umax;
    float* my_stream;
    float* FO;  // output planes at band row 0 (image row y0 - (K-1))
    float* BO;
    int opitch;
};

// Records and image value of slot k's pixel of step tr + 1 (c = the ring
// column of step tr).
template <int K>
__device__ __forceinline__ CoefR load_coef(const ChainCtx<K>& x_, int c, int k) {
    using Gm = Geom<K>;
    const int dp = 1 - k + Gm::SH;
    const int row = K - 1 - k;
    const int ri = x_.rb + 4 * (c + row * Gm::RS + dp);
    const float4 wa = lds4(Gm::REC_A + ri);
    const float4 wb = lds4(Gm::REC_B + ri);
    CoefR co;
    co.dL = wa.x;
    co.dD = wa.y;
    co.dR = wa.z;
    co.dU = wa.w;
    co.iS = wb.x;
    co.u = pk2(wb.y, __fsub_rn(1.0f, wb.y));
    co.pq = pk2(wb.z, wb.w);
    co.I = lds(x_.lb + c + Gm::C_I + row * Gm::RS + dp);
    return co;
}

template <int K>
struct GroupAddr {
    float* fo;    // flush address of step 0, F plane
    float* bo;
    int o0;       // output-ring float index of step 0
    bool seg_ok;  // the segment start column is inside the row
    int jf0;      // flushed band row of step 0
    float* sdst;  // lane 31's boundary-stream slot of step 0
};
// With K = 2 (mod 4) a group's four flushed rows never cross a 16-row half
// of the band: step s of the group flushes row jf0 + s of segment xs0.
template <int K>
__device__ __forceinline__ constexpr bool group_addr_ok() { return K % 4 == 2; }

template <int K, int CK>
__device__ __forceinline__ GroupAddr<K> group_addr(const ChainCtx<K>& x_, int t4) {
    using Gm = Geom<K, CK>;
    constexpr int SEG = Gm::SEG;
    GroupAddr<K> g;
    const int lane = x_.lane;
    const int col = lane & (SEG - 1);
    const int u0 = t4 - (K - 1) - (SEG - 1);
    g.jf0 = (u0 & (SEG - 1)) + (lane & 16);
    const int xs0 = (u0 & ~(SEG - 1)) - (lane & 16);
    g.seg_ok = xs0 >= 0;
    const unsigned off = unsigned(g.jf0 * x_.opitch + xs0 + col);  // (used only when seg_ok)
    g.fo = x_.FO + off;
    g.bo = x_.BO + off;
    g.o0 = x_.cb + Gm::C_O + g.jf0 * Gm::OW + (xs0 & SEG) + col;
    g.sdst = x_.my_stream + (long long)(t4 - 31) * K * 2;
    return g;
}

// One wavefront step of a chain warp: no barrier inside.  G: a pixel of this
// step may be on the image border (clamped neighbours).  YU / YD (G false):
// interior columns of a band touching row 0 / row h-1 (the first band heads
// every chain: it pays for the U clamp only).  XL (G false): the first steps
// of a band (x <= 0 only).
template <int K, bool G, int CK, bool YU = false, bool YD = false, bool XL = false>
__device__ __forceinline__ void chain_step(LaneState<K>& st, const ChainCtx<K>& x_, int tr,
                                           const GroupAddr<K>* ga = nullptr, int gs = 0) {
    constexpr bool Y = YU || YD;
    using Gm = Geom<K, CK>;
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
        const int cn = x_.cb + Gm::C_C + (tr % CK) * K * 2;
#pragma unroll
        for (int k = 0; k < K; ++k) recv[k] = make_float2(lds(cn + 2 * k), lds(cn + 2 * k + 1));
    }

    float2 nv[K];
    const int xs0 = tr - lane;  // slot-0 column
#pragma unroll
    for (int k = 0; k < K; ++k) {
        float2 L = st.outp[k], U = recv[k], R, D;
        if (k == 0) {
            R = make_float2(lds(rc + Gm::C_F + 1 + Gm::SH), lds(rc + Gm::C_B + 1 + Gm::SH));
            D = make_float2(lds(rc + Gm::C_F + Gm::RS + Gm::SH), lds(rc + Gm::C_B + Gm::RS + Gm::SH));
        } else {
            R = recv[k - 1];
            D = st.outp[k - 1];
        }
        if (G || Y || XL) {
            const int x = xs0 - k, y = y0 + lane - k;
            const float2 self = k == 0 ? make_float2(lds(rc + Gm::C_F + Gm::SH), lds(rc + Gm::C_B + Gm::SH))
                                       : st.rprev[k > 0 ? k - 1 : 0];
            if (G || XL) {
                if (!(x > 0)) L = self;
            }
            if (G) {
                if (!(x < w - 1)) R = self;
            }
            if (G || YU) {
                if (!(y > 0)) U = self;
            }
            if (G || YD) {
                if (!(y < h - 1)) D = self;
            }
        }
        nv[k] = pixel_applyr(st.co[k], L, R, U, D);
    }

    // the next step's records (published by the producer at least a group ago)
#pragma unroll
    for (int k = 0; k < K; ++k) st.co[k] = load_coef<K>(x_, c, k);

    // output ring (last sweep only): column x mod 32 == c
    {
        bool ok = true;
        if (G) {
            const int x = xs0 - (K - 1);
            ok = x >= 0 && x < w && y0 + lane - (K - 1) >= 0 && y0 + lane - (K - 1) < h;
        }
        if (ok) {  // (Y: rows outside the image land in the ring but are never flushed)
            const int o = x_.cb + Gm::C_O + lane * Gm::OW + c;
            sts(o, nv[K - 1].x);
            sts(o + Gm::OPL, nv[K - 1].y);
        }
    }

    // boundary stream for the band below: lane 31's K outputs of this step
    if (x_.has_down && lane == kRows - 1 && (!(G || XL) || (tr - 31 >= 0 && tr - 31 < x_.Umax))) {
        float* dst = (!G && group_addr_ok<K>() && ga) ? ga->sdst + gs * K * 2 : x_.my_stream + size_t(tr - 31) * K * 2;
        if (K % 2 == 0) {
#pragma unroll
            for (int k = 0; k + 1 < K; k += 2)
                st_relaxed_v4(dst + 2 * k, make_float4(nv[k].x, nv[k].y, nv[k + 1].x, nv[k + 1].y));
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) st_relaxed_v2(dst + 2 * k, nv[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (G || Y || XL) st.rprev[k] = recv[k];
        st.outp[k] = nv[k];
    }
}

// Flush the 16-column output row segments completed at step tr: rows jf
// (lanes 0-15) and jf+16 (lanes 16-31), one coalesced 64-byte store per plane
// each.  Called once per group after a __syncwarp: the 32-column ring keeps a
// completed segment for 16 more steps.
template <int K, bool G, int CK, bool Y = false, bool XL = false>
__device__ __forceinline__ void flush_step(const ChainCtx<K>& x_, int tr, const GroupAddr<K>* ga = nullptr,
                                           int gs = 0) {
    using Gm = Geom<K, CK>;
    constexpr int SEG = Gm::SEG;
    const int lane = x_.lane, y0 = x_.y0, w = x_.w, h = x_.h;
    if (!G && group_addr_ok<K>() && ga) {
        bool ok = true;
        if (Y) {
            const int yf = y0 + ga->jf0 + gs - (K - 1);
            ok = yf >= 0 && yf < h;
        }
        if (XL) ok = ok && ga->seg_ok;
        if (ok) {
            const long long ro = (long long)gs * x_.opitch;
            const int o = ga->o0 + gs * Gm::OW;
            stg(ga->fo + ro, lds(o));
            stg(ga->bo + ro, lds(o + Gm::OPL));
        }
    } else {
        const int col = lane & (SEG - 1);
        const int u = tr - (K - 1) - (SEG - 1);
        const int jf = (u & (SEG - 1)) + (lane & 16);
        const int xs = (u & ~(SEG - 1)) - (lane & 16);  // segment start column
        bool ok = true;
        if (G) {
            const int yf = y0 + jf - (K - 1);
            ok = xs >= 0 && xs + SEG - 1 < w && yf >= 0 && yf < h;
        } else {
            if (Y) {
                const int yf = y0 + jf - (K - 1);
                ok = yf >= 0 && yf < h;
            }
            if (XL) ok = ok && xs >= 0;
        }
        if (ok) {
            const unsigned off = unsigned(jf * x_.opitch + xs + col);
            const int o = x_.cb + Gm::C_O + jf * Gm::OW + (xs & SEG) + col;
            stg(x_.FO + off, lds(o));
            stg(x_.BO + off, lds(o + Gm::OPL));
        }
        if (G && ((w - 1) & (SEG - 1)) != SEG - 1) {  // partial last segment of a row
            const int je = tr - (K - 1) - (w - 1);
            const int x0 = (w - 1) & ~(SEG - 1);
            const int ye = y0 + je - (K - 1);
            if (je >= 0 && je < 32 && ye >= 0 && ye < h && lane < w - x0) {
                const unsigned off = unsigned(je * x_.opitch + x0 + lane);
                const int o = x_.cb + Gm::C_O + je * Gm::OW + (x0 & SEG) + lane;
                stg(x_.FO + off, lds(o));
                stg(x_.BO + off, lds(o + Gm::OPL));
            }
        }
    }
}

#ifndef FGM_REPOLL
#define FGM_REPOLL 1
#endif
#ifdef FGM_WS_TRACE  // development probe: cycles per phase of a warp
#define TR_DECL long long tr_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tr_t = clock64(), tr_start = tr_t
#define TR(i)                           \
    {                                   \
        const long long c_ = clock64(); \
        tr_[i] += c_ - tr_t;            \
        tr_t = c_;                      \
    }
#else
#define TR_DECL
#define TR(i)
#endif

// What the three warps of a channel and the producers share about a band.
template <int K, int CK>
struct BandGeo {
    using Gm = Geom<K, CK>;
    int w, h, y0, Umax, tend, ngroups;
    bool yband, ytop;
    int fast_lo, fast_hi;
    __device__ __forceinline__ BandGeo(const SweepJob& J, int q) {
        w = J.w;
        h = J.h;
        y0 = q * kRows;
        Umax = w + K - 1;
        tend = 31 + Umax;  // lane 31's last column is Umax - 1
        ngroups = (tend + Gm::S + Gm::S - 1) / Gm::S;  // groups t4 = -S, 0, S, ...
        yband = y0 - (K - 1) <= 0 || y0 + 31 >= h - 1;
        ytop = y0 + 31 < h - 1;  // (with yband: the band touches row 0 only)
        fast_lo = 32 + K;  // a step tr has no column border iff fast_lo <= tr < fast_hi
        fast_hi = w - 2;
    }
};

template <int K>
__device__ __forceinline__ ChainCtx<K> make_ctx(const SweepJob& J, int q, int ch, int lane, int fault) {
    using Gm = Geom<K>;
    const int y0 = q * kRows;
    const size_t slen = sweep_stream_len(J.w, K);
    ChainCtx<K> cx;
    cx.cb = ch * Gm::CHSZ;
    cx.lb = cx.cb + lane * Gm::RS;
    cx.rb = 4 * lane * Gm::RS;
    cx.lane = lane;
    cx.y0 = y0;
    cx.w = J.w;
    cx.h = J.h;
    cx.has_up = q > 0;
    cx.has_down = q < J.nb - 1 && !(fault == 1 && q == 0);  // (fault 1: band 0 never publishes)
    cx.Umax = J.w + K - 1;
    cx.my_stream = J.stream + size_t(q * 3 + ch) * slen;
    // band-relative output base (row y0 - (K-1) may be negative for the first
    // band: only the pointer arithmetic goes there, stores are bounds-checked)
    cx.FO = J.fg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    cx.BO = J.bg_out + (long long)ch * J.ostride + (long long)(y0 - (K - 1)) * J.opitch;
    cx.opitch = J.opitch;
    return cx;
}

// Chain warp of channel ch: the recurrence only.  Group n starts once the
// channel's helper has the group's ring data in shared memory and the
// producers have finished groups n and n + 1.  Returns false when the launch
// was aborted.
template <int K, int CK>
__device__ __forceinline__ bool run_chain(const SweepJob& J, int q, int ch, int lane, unsigned sbase, const SweepFail& F,
                                          int fault) {
    using Gm = Geom<K, CK>;
    const BandGeo<K, CK> bg(J, q);
    const int Umax = bg.Umax;
    const ChainCtx<K> cx = make_ctx<K>(J, q, ch, lane, fault);
    const float* up_stream = q > 0 ? J.stream + size_t((q - 1) * 3 + ch) * sweep_stream_len(J.w, K) : nullptr;
    const unsigned pr = sbase + 4u * unsigned(Gm::OFF_PR);
    const unsigned pr_mine = pr + 4u * unsigned(Gm::PR_CHAIN + ch), pr_load = pr + 4u * unsigned(Gm::PR_LOAD + ch);

    LaneState<K> st;
#pragma unroll
    for (int k = 0; k < K; ++k) st.outp[k] = st.rprev[k] = make_float2(0.0f, 0.0f);

    constexpr int S = Gm::S;
    constexpr int t0 = -S;
    float4 pend = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool lane_ch = lane < Gm::CH4;
    bool pend_ok = false;
    if (cx.has_up && lane_ch) pend = ld_relaxed_v4(up_stream + 4 * lane);

    int prod0 = 0, prod1 = 0;  // cached producer progress (iterations finished by producer 0 / 1)
    int loaded = 0;            // cached helper progress (groups whose ring data is in shared memory)
    int n = 0;
    TR_DECL;
#ifdef FGM_WS_TRACE
    unsigned long long tl_[6] = {global_ns(), 0, 0, 0, 0, 0};
#endif
    for (int t4 = t0; t4 < bg.tend; t4 += S, ++n) {
        TR(0);
#ifdef FGM_WS_TRACE
        if (n == 1) tl_[1] = global_ns();   // before group t4 = 0
        if (n == 2) tl_[2] = global_ns();   // after group t4 = 0
        if (n == 10) tl_[3] = global_ns();  // after step 35
        if (n == 100) tl_[4] = global_ns();
        if (n == 200) tl_[5] = global_ns();
#endif
        if (loaded < n + 1) {
            loaded = wait_progress(pr_load, n + 1, lane, F);
            if (loaded < 0) return false;
        }
        TR(1);
        // the records of this group and of the next group's first step: the
        // groups <= g1, of which producer 0 computes the even ones
        {
            const int g1 = min(n + 1, bg.ngroups - 1);
            const int need0 = g1 / 2 + 1, need1 = (g1 + 1) / 2;
            if (prod0 < need0) {
                prod0 = wait_progress(pr + 4u * unsigned(Gm::PR_PROD), need0, lane, F);
                if (prod0 < 0) return false;
            }
            if (prod1 < need1) {
                prod1 = wait_progress(pr + 4u * unsigned(Gm::PR_PROD + 1), need1, lane, F);
                if (prod1 < 0) return false;
            }
        }
        __syncwarp();
        TR(2);
        if (t4 < 0) {
            const int c = (-1 - lane - Gm::SH) & (Gm::RW - 1);
#pragma unroll
            for (int k = 0; k < K; ++k) st.co[k] = load_coef<K>(cx, c, k);
        } else {
            if (cx.has_up && t4 < Umax) {
                const int nxt = (t4 & ~(CK - 1)) + CK;
                if ((t4 % CK) == 0) {
                    if (!acquire_chunk<K, CK>(pend, up_stream, t4, Umax, lane, cx.cb + Gm::C_C, F)) return false;
                    pend_ok = false;
                    if (nxt < Umax && lane_ch) pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
                } else if (FGM_REPOLL && !pend_ok && nxt < Umax) {
                    pend_ok = __all_sync(kFull, chunk_complete<K, CK>(pend, nxt, Umax, lane));
                    if (!pend_ok && lane_ch) pend = ld_relaxed_v4(up_stream + size_t(nxt) * K * 2 + 4 * lane);
                }
                __syncwarp();
            }
            TR(3);
            // (block order: the cold variants first; the interior block and, last,
            // the first band's -- the band that paces every other -- fall through
            // to the group's tail)
            const bool xin = t4 >= bg.fast_lo && t4 + S <= bg.fast_hi;
            if (!xin) {
                if (t4 < bg.fast_lo && t4 + S <= bg.fast_hi) {  // band start: left border only
                    const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
                    if (bg.yband) {
#pragma unroll
                        for (int s = 0; s < S; ++s) chain_step<K, false, CK, true, true, true>(st, cx, t4 + s, &ga, s);
                    } else {
#pragma unroll
                        for (int s = 0; s < S; ++s) chain_step<K, false, CK, false, false, true>(st, cx, t4 + s, &ga, s);
                    }
                } else {
#pragma unroll 1
                    for (int s = 0; s < S; ++s) chain_step<K, true, CK>(st, cx, t4 + s);
                }
            } else if (bg.yband && !bg.ytop) {
                const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll
                for (int s = 0; s < S; ++s) chain_step<K, false, CK, true, true>(st, cx, t4 + s, &ga, s);
            } else if (!bg.yband) {
                const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll
                for (int s = 0; s < S; ++s) chain_step<K, false, CK>(st, cx, t4 + s, &ga, s);
            } else {  // the first band of a taller image: U clamps only
                const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll
                for (int s = 0; s < S; ++s) chain_step<K, false, CK, true, false>(st, cx, t4 + s, &ga, s);
            }
        }
        TR(4);
        __syncwarp();  // every lane's output-ring stores and ring / record reads of the group are issued
        if (lane == 0) st_volatile_cta(pr_mine, n + 1);
        TR(5);
    }
#ifdef FGM_WS_TRACE
    if (lane == 0 && ch == 0 && (q <= 3 || q == J.nb / 2))
        printf("timeline band %d: launch +0, before g0 %llu ns, after g0 %llu, after step 35 %llu, n=100 %llu, n=200 %llu, end %llu\n", q,
               tl_[1] - tl_[0], tl_[2] - tl_[0], tl_[3] - tl_[0], tl_[4] - tl_[0], tl_[5] - tl_[0], global_ns() - tl_[0]);
    if (lane == 0 && ch == 0 && (q == 0 || q == 1 || q == J.nb / 2 || q == J.nb - 1))
        printf("chain %d/%d K=%d w=%d groups %d: total %lld cyc | loop %lld loadwait %lld prodwait %lld chunk %lld steps %lld "
               "publish %lld\n",
               q, J.nb, K, J.w, n, clock64() - tr_start, tr_[0], tr_[1], tr_[2], tr_[3], tr_[4], tr_[5]);
#endif
    return true;
}

// Helper warp of channel ch: streams the channel's I_c / F_c / B_c rows into
// the rings ahead of the chain warp and flushes its output rows behind it.
// Iteration i first publishes the ring data of chain group i + 1 (the blocks
// issued M - 1 iterations earlier have landed: nothing the chain warp waits
// for depends on the rest of the iteration); then, once the chain warp has
// finished group i - 1, it issues the ring blocks "of the end of group i" (they
// overwrite columns last read in group i - 1) and flushes group i - 1's
// completed output segments.
template <int K, bool V4, int CK>
__device__ __forceinline__ bool run_helper(const SweepJob& J, int q, int ch, int lane, unsigned sbase, const SweepFail& F,
                                           int fault) {
    using Gm = Geom<K, CK>;
    const BandGeo<K, CK> bg(J, q);
    const int w = bg.w;
    const ChainCtx<K> cx = make_ctx<K>(J, q, ch, lane, fault);
    const unsigned cbase = sbase + 4u * unsigned(cx.cb);
    const RowSrc own = make_rowsrc<K>(J, ch, bg.y0, lane, true, true, cbase);
    const bool has_x = lane >= 33 - K || lane == 0;
    const RowSrc ext = make_rowsrc<K>(J, ch, bg.y0, lane == 0 ? 32 : lane - 32, lane >= 33 - K, lane == 0, cbase);
    const FlatSrc<K> flat = make_flat<K>(J, ch, bg.y0, lane, cbase);
    const unsigned pr = sbase + 4u * unsigned(Gm::OFF_PR);
    const unsigned pr_chain = pr + 4u * unsigned(Gm::PR_CHAIN + ch), pr_mine = pr + 4u * unsigned(Gm::PR_LOAD + ch);

    constexpr int S = Gm::S;
    constexpr int t0 = -S;
    prologue_row<K, V4>(own, t0, w);
    if (has_x) prologue_row<K, V4>(ext, t0, w);
    cp_commit();
#pragma unroll
    for (int i = 1; i < Gm::M; ++i) cp_commit();

    // groups whose issued blocks are inside [0, w) for every row -K .. 32
    const int issue_lo = 32 - Gm::L, issue_hi = w - 2 * S - Gm::L - K;
    int chain_done = 0;
    // flush the output segments completed in group t4 (all of whose steps are done)
    auto flush_group = [&](int t4) {
        if (t4 < 0) return;
        const bool xin = t4 >= bg.fast_lo && t4 + S <= bg.fast_hi;
        if (xin && !bg.yband) {
            const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll 1
            for (int s = 0; s < S; ++s) flush_step<K, false, CK>(cx, t4 + s, &ga, s);
        } else if (xin) {
            const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll 1
            for (int s = 0; s < S; ++s) flush_step<K, false, CK, true>(cx, t4 + s, &ga, s);
        } else if (t4 < bg.fast_lo && t4 + S <= bg.fast_hi) {  // band start: segments left of column 0 are skipped
            const GroupAddr<K> ga = group_addr<K, CK>(cx, t4);
#pragma unroll 1
            for (int s = 0; s < S; ++s) flush_step<K, false, CK, true, true>(cx, t4 + s, &ga, s);
        } else {
#pragma unroll 1
            for (int s = 0; s < S; ++s) flush_step<K, true, CK>(cx, t4 + s);
        }
    };
    int i = 0;
    for (int t4 = t0; t4 < bg.tend; t4 += S, ++i) {
        // first, what the chain warp may be waiting for: the blocks issued M - 1
        // iterations ago have landed -- the ring data of chain group i + 1
        cp_wait<Gm::M - 2>();
        __syncwarp();
        if (lane == 0) st_volatile_cta(pr_mine, i + 2);
        if (chain_done < i) {
            chain_done = wait_progress(pr_chain, i, lane, F);
            if (chain_done < 0) {
                cp_wait<0>();
                return false;
            }
        }
        __syncwarp();
        if (V4 && t4 >= issue_lo && t4 < issue_hi) {  // (rows outside the image: a clamped row, never read unclamped)
            issue_flat<K>(flat, t4);
        } else if (V4 && t4 < issue_hi) {  // the band's first groups: every band's start is on the critical path
            issue_flat<K, true>(flat, t4);
        } else {
            issue_row<K, V4>(own, t4, w);
            if (has_x) issue_row<K, V4>(ext, t4, w);
        }
        cp_commit();
        flush_group(t4 - S);
    }
    chain_done = wait_progress(pr_chain, i, lane, F);
    cp_wait<0>();
    if (chain_done < 0) return false;
    __syncwarp();
    flush_group(t0 + (i - 1) * S);
    return true;
}

// ---- producer warps -----------------------------------------------------------

template <bool V4>
__device__ __forceinline__ void put_alpha(const float* g, unsigned srow, int x0, int w, int aw_mask) {
    if (!g || x0 < 0 || x0 >= w) return;
    const int n = min(w - x0, 4);
    const unsigned d = srow + 4u * unsigned(x0 & aw_mask);
    if (V4) {
        cp_async16(d, g + x0, 4 * n);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) cp_async4(d + 4 * i, i < n ? g + x0 + i : g, i < n ? 4 : 0);
    }
}

// Store the record of pixel (x, band row r): record row r + K - 1.
template <int K, int CK>
__device__ __forceinline__ void store_record(const CoefR& co, float a, int r, int x, bool on) {
    using Gm = Geom<K, CK>;
    const float2 pq = upk2(co.pq);
    const int col = x & (Gm::RW - 1);
    const int ri = 4 * ((r + K - 1) * Gm::RS + col);
    const float4 wa = make_float4(co.dL, co.dD, co.dR, co.dU), wb = make_float4(co.iS, a, pq.x, pq.y);
    if (on) {
        sts4(Gm::REC_A + ri, wa);
        sts4(Gm::REC_B + ri, wb);
        if (col < Gm::MIR) {
            sts4(Gm::REC_A + ri + 4 * Gm::RW, wa);
            sts4(Gm::REC_B + ri + 4 * Gm::RW, wb);
        }
    }
}

// The records of producer times t4 .. t4 + S - 1.  Lane r computes pixels
// (t - r, band row r) for the S times t, carrying a and the right edge weight
// along the row (the left edge weight of a pixel is the right edge weight of
// its left neighbour: |a - b| is exactly symmetric); K > 1: lane l < S (K - 1)
// also computes pixel (t4 + l % S - i, band row -i), i = 1 + l / S, once per
// group.  GX / GY: clamp the column / row neighbours at the image border (a
// clamped neighbour is the pixel itself: edge weight eps,
// multilevel.cpp:104-106).  `al`: float index of this producer's alpha ring.
template <int K, bool GX, bool GY, int CK>
__device__ __forceinline__ void produce_group(int al, int t4, int lane, int y0, int w, int h, float eps, float omega) {
    using Gm = Geom<K, CK>;
    constexpr int AM = Gm::AW - 1;
    {
        const int ca = al + (lane + K) * Gm::ARS;
        const int y = y0 + lane;
        int x = t4 - lane;
        float a = lds(ca + (x & AM));
        float dL = edge_weight(a, lds(ca + ((x - 1) & AM)), eps, omega);
#pragma unroll
        for (int s = 0; s < Gm::S; ++s, ++x) {
            const float an = lds(ca + ((x + 1) & AM));
            float aR = an, aU = lds(ca - Gm::ARS + (x & AM)), aD = lds(ca + Gm::ARS + (x & AM));
            if (GX) {
                if (x <= 0) dL = eps;
                if (x >= w - 1) aR = a;
            }
            if (GY) {
                if (y <= 0) aU = a;
                if (y >= h - 1) aD = a;
            }
            const CoefR co = pixel_coefr_dl(a, dL, aR, aU, aD, 0.0f, eps, omega);
            store_record<K, CK>(co, a, lane, x, true);
            a = an;
            dL = co.dR;
        }
    }
    if (K > 1) {
        const bool on = lane < Gm::S * (K - 1);
        const int i = on ? 1 + lane / Gm::S : 1;
        const int x = t4 + (lane % Gm::S) - i, y = y0 - i;
        const int ca = al + (K - i) * Gm::ARS;
        const float a = lds(ca + (x & AM));
        float aL = lds(ca + ((x - 1) & AM)), aR = lds(ca + ((x + 1) & AM));
        float aU = lds(ca - Gm::ARS + (x & AM)), aD = lds(ca + Gm::ARS + (x & AM));
        if (GX) {
            if (x <= 0) aL = a;
            if (x >= w - 1) aR = a;
        }
        if (GY) {
            if (y <= 0) aU = a;
            if (y >= h - 1) aD = a;
        }
        const CoefR co = pixel_coefr_dl(a, edge_weight(a, aL, eps, omega), aR, aU, aD, 0.0f, eps, omega);
        store_record<K, CK>(co, a, -i, x, on);
    }
}

// Producer pw (0 / 1) computes the groups n = pw (mod 2) from its own alpha
// ring.  Group n may start once every chain warp works on group >= n - kAhead
// (its record slots were last read in group n - 6).
template <int K, bool V4, int CK>
__device__ __forceinline__ bool run_producer(const SweepJob& J, int q, int pw, int lane, unsigned sbase, float eps,
                                             float omega, const SweepFail& F) {
    using Gm = Geom<K, CK>;
    const BandGeo<K, CK> bg(J, q);
    const int w = bg.w, h = bg.h, y0 = bg.y0;
    constexpr int S = Gm::S;
    constexpr int t0 = -S;
    const int al = Gm::OFF_AL + pw * Gm::NA * Gm::ARS;

    // alpha rows this lane streams: band row `lane` and, lanes 0..K, one of
    // the rows -K..-1, 32
    const bool has_e = lane <= K;
    const int er = lane < K ? lane - K : 32;
    const int yo = y0 + lane, ye = y0 + er;
    const float* g_own = yo < h ? J.alpha + (long long)yo * J.ipitch : nullptr;
    const float* g_ext = has_e && ye >= 0 && ye < h ? J.alpha + (long long)ye * J.ipitch : nullptr;
    const unsigned s_own = sbase + 4u * unsigned(al + (lane + K) * Gm::ARS);
    const unsigned s_ext = sbase + 4u * unsigned(al + (er + K) * Gm::ARS);
    const unsigned pr = sbase + 4u * unsigned(Gm::OFF_PR);
    const unsigned pr_mine = pr + 4u * unsigned(Gm::PR_PROD + pw);

    // an iteration covers 2S producer times: two S-column blocks per row
    const int tfirst = t0 + pw * S;
    for (int x0 = 0; x0 <= ((tfirst - S + Gm::LA - lane) & ~(S - 1)); x0 += S) put_alpha<V4>(g_own, s_own, x0, w, Gm::AW - 1);
    for (int x0 = 0; x0 <= ((tfirst - S + Gm::LA - er) & ~(S - 1)); x0 += S) put_alpha<V4>(g_ext, s_ext, x0, w, Gm::AW - 1);
    cp_commit();
#pragma unroll
    for (int i = 1; i < Gm::MA; ++i) cp_commit();

    int chain_at = 0;  // cached min over the chain warps of their finished groups
    int it = 0;
    TR_DECL;
    for (int n = pw; n < bg.ngroups; n += 2, ++it) {
        const int t4 = t0 + n * S;
        TR(0);
        if (n - kAhead > chain_at) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int v = wait_progress(pr + 4u * unsigned(Gm::PR_CHAIN + c), n - kAhead, lane, F);
                if (v < 0) {
                    cp_wait<0>();
                    return false;
                }
                chain_at = c == 0 ? v : min(chain_at, v);
            }
        }
        TR(1);
        cp_wait<Gm::MA - 1>();
        __syncwarp();
        TR(2);
        const bool xin = t4 - 31 >= 1 && t4 + S - 1 <= w - 2;  // every pixel of the group has both column neighbours
        if (xin && !bg.yband)
            produce_group<K, false, false, CK>(al, t4, lane, y0, w, h, eps, omega);
        else if (xin)
            produce_group<K, false, true, CK>(al, t4, lane, y0, w, h, eps, omega);
        else
            produce_group<K, true, true, CK>(al, t4, lane, y0, w, h, eps, omega);
        TR(3);
        __syncwarp();  // every lane's records are issued, every lane's alpha reads are done
        {
            const int b_own = (t4 + S + Gm::LA - lane) & ~(S - 1), b_ext = (t4 + S + Gm::LA - er) & ~(S - 1);
            put_alpha<V4>(g_own, s_own, b_own - S, w, Gm::AW - 1);
            put_alpha<V4>(g_own, s_own, b_own, w, Gm::AW - 1);
            if (has_e) {
                put_alpha<V4>(g_ext, s_ext, b_ext - S, w, Gm::AW - 1);
                put_alpha<V4>(g_ext, s_ext, b_ext, w, Gm::AW - 1);
            }
        }
        cp_commit();
        if (lane == 0) st_volatile_cta(pr_mine, it + 1);
        TR(4);
    }
#ifdef FGM_WS_TRACE
    if (lane == 0 && pw == 0 && (q == 0 || q == 1 || q == J.nb / 2))
        printf("producer %d/%d K=%d iterations %d: total %lld cyc | loop %lld chainwait %lld cpwait %lld produce %lld issue %lld\n",
               q, J.nb, K, it, clock64() - tr_start, tr_[0], tr_[1], tr_[2], tr_[3], tr_[4]);
#endif
    cp_wait<0>();
    __syncwarp();
    return true;
}

struct SweepArgs {
    const SweepJob* jobs;
    const int2* order;  // (job, band * 3 + channel) per item, three items per band
    int total_bands;
    unsigned* ticket;
    float eps, omega;
    SweepFail fail;
    int fault;
};

// Warp roles of a band CTA.  Schedulers serve warp w % 4 and prefer the higher
// warp id: warps 5-7 are the chain warps of channels 0-2 (one scheduler each,
// with priority), warps 1-3 their helpers on the same schedulers (they fill
// the chain warps' stall slots), warps 0 and 4 the producers (the fourth
// scheduler).
constexpr int kWsThreads = 256;

template <int K, bool V4, int CK>
__device__ __forceinline__ void run_band_cta(const SweepJob& J, int q, int warp, int lane, unsigned sbase,
                                             const SweepArgs& A) {
    if ((warp & 3) == 0)
        run_producer<K, V4, CK>(J, q, warp >> 2, lane, sbase, A.eps, A.omega, A.fail);
    else if (warp > 4)
        run_chain<K, CK>(J, q, warp - 5, lane, sbase, A.fail, A.fault);
    else
        run_helper<K, V4, CK>(J, q, warp - 1, lane, sbase, A.fail, A.fault);
}

template <int K, int CK>
__global__ void __launch_bounds__(kWsThreads, 1) sweep_ws_kernel(SweepArgs A) {
    using Gm = Geom<K, CK>;
    __shared__ unsigned s_tk;
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(ws_sm4));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) {
            unsigned tk = atomicAdd(A.ticket, 1u);
            if (*reinterpret_cast<volatile int*>(A.fail.abort_flag)) tk = 0xffffffffu;
            s_tk = tk;
#pragma unroll
            for (int i = 0; i < Gm::NPR; ++i) reinterpret_cast<int*>(smf())[Gm::OFF_PR + i] = 0;
        }
        __syncthreads();
        const unsigned tk = s_tk;
        if (tk >= unsigned(A.total_bands)) return;
        const int2 jb = A.order[3 * tk];  // (job, band * 3)
        const SweepJob J = A.jobs[jb.x];
        if (!J.vec4)
            run_band_cta<K, false, CK>(J, jb.y / 3, warp, lane, sbase, A);
        else
            run_band_cta<K, true, CK>(J, jb.y / 3, warp, lane, sbase, A);
        __syncthreads();  // every warp is done with the band's shared memory (and has read s_tk)
    }
}

template <int K>
cudaError_t ws_grid_cap(int& cap) {
    static PerDevice<int> cfg;
    return cfg.get(cap, [](int dev, int& v) {
        const int sm4 = int(Geom<K, 4>::TOTAL * sizeof(float)), sm16 = int(Geom<K, kChunk>::TOTAL * sizeof(float));
        cudaError_t e = cudaFuncSetAttribute(sweep_ws_kernel<K, kChunk>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm16);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_ws_kernel<K, kChunk>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_ws_kernel<K, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(sweep_ws_kernel<K, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int sms = 0, per_sm = 0;
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_ws_kernel<K, kChunk>, kWsThreads, size_t(sm16));
        v = std::max(1, sms * std::max(1, per_sm));
        return e;
    });
}

// Launches whose bands all fit on the GPU at once poll 4-column boundary
// chunks (a shorter hand-over lag on the critical path), the others 16.
template <int K>
cudaError_t launch_ws_k(const SweepArgs& A, cudaStream_t s) {
    int cap = 0;
    cudaError_t e = ws_grid_cap<K>(cap);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(A.total_bands, cap));
    if (A.total_bands <= cap)
        sweep_ws_kernel<K, 4><<<grid, kWsThreads, size_t(Geom<K, 4>::TOTAL) * sizeof(float), s>>>(A);
    else
        sweep_ws_kernel<K, kChunk><<<grid, kWsThreads, size_t(Geom<K, kChunk>::TOTAL) * sizeof(float), s>>>(A);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_sweep_ws(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket,
                            float eps, float omega, int* abort_flag, int* fault_count, cudaStream_t s) {
    SweepArgs A;
    A.jobs = jobs_dev;
    A.order = order_dev;
    A.total_bands = total_items / 3;
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
