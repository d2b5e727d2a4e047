// sm_100a kernels of the multi-level F/B estimator.
//
//   K1/K2 resample_kernel  -- bilinear level resampling (image.cpp:71-133)
//   K4    coarse_kernel    -- all coarse levels of an image in one CTA, in
//                             shared memory, exact Gauss-Seidel order
//   (K3, the big-level sweep, lives in sweep.cu)
//
// See DESIGN.md for the dependency analysis that makes K3 exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "fgm_device.cuh"
#include "fgm_internal.h"

namespace fgm {

// ============================================================================
// K1/K2: resample.  One CTA row-loop per destination row, threads along x
// (coalesced stores).  Equal sizes are an unclamped copy (image.cpp:116,127).
// ============================================================================
// Tiles of 128 columns x kResRows rows: each thread keeps its column's x-tap
// (fp64, once) for all rows of the tile; the tile's y-taps are computed once
// into shared memory; every plane's four taps are loaded before any lerp.
constexpr int kResCols = 128;
constexpr int kResRows = 8;

// Index type Ix: int when every element index of the job fits in 32 bits
// (one IMAD.WIDE per address instead of 64-bit arithmetic), else long long.
template <int NP, typename Ix>
__device__ __forceinline__ void resample_tile(const ResampleJob& J, int x, int ybase, const Tap* tys) {
    if (x >= J.dw) return;
    const int yend = min(kResRows, J.dh - ybase);
    const float* __restrict__ src = J.src;
    float* __restrict__ dst = J.dst;
    const Ix sps = Ix(J.spstride), dps = Ix(J.dpstride), sp = Ix(J.spitch), dp = Ix(J.dpitch);
    Ix o = Ix(ybase) * dp + x;
    if (J.sw == J.dw && J.sh == J.dh) {  // resize to the same size: unclamped copy
        Ix is = Ix(ybase) * sp + x;
        for (int r = 0; r < yend; ++r, is += sp, o += dp) {
            float v[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) v[p] = __ldg(src + (p * sps + is));
#pragma unroll
            for (int p = 0; p < NP; ++p) dst[p * dps + o] = v[p];
        }
        return;
    }
    const Tap tx = make_tap_s(x, J.sw, J.sx);
    const int dx = tx.i1 - tx.i0;
    for (int r = 0; r < yend; ++r, o += dp) {
        const Tap ty = tys[r];
        const Ix a0 = Ix(ty.i0) * sp + tx.i0, c0 = Ix(ty.i1) * sp + tx.i0;
        float v[NP][4];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float* s = src + p * sps;
            v[p][0] = __ldg(s + a0);
            v[p][1] = __ldg(s + a0 + dx);
            v[p][2] = __ldg(s + c0);
            v[p][3] = __ldg(s + c0 + dx);
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) dst[p * dps + o] = bilerp(v[p][0], v[p][1], v[p][2], v[p][3], tx.t, ty.t);
    }
}

__device__ __forceinline__ void resample_tile_generic(const ResampleJob& J, int x, int ybase, const Tap* tys) {
    if (x >= J.dw) return;  // generic plane count (fgm_resize_f32)
    const int yend = min(kResRows, J.dh - ybase);
    const bool ident = J.sw == J.dw && J.sh == J.dh;
    const Tap tx = make_tap_s(x, J.sw, J.sx);
    for (int r = 0; r < yend; ++r) {
        const long long o = (long long)(ybase + r) * J.dpitch + x;
        const long long so = (long long)(ybase + r) * J.spitch + x;
        const Tap ty = tys[r];
        const long long r0 = (long long)ty.i0 * J.spitch, r1 = (long long)ty.i1 * J.spitch;
        for (int p = 0; p < J.nplanes; ++p) {
            const float* s = J.src + p * J.spstride;
            J.dst[p * J.dpstride + o] =
                ident ? s[so] : bilerp(s[r0 + tx.i0], s[r0 + tx.i1], s[r1 + tx.i0], s[r1 + tx.i1], tx.t, ty.t);
        }
    }
}

// Persistent blocks walk the flat tile space of all jobs of the launch.
__global__ void __launch_bounds__(kResCols) resample_kernel(const ResampleJob* __restrict__ jobs, int njobs,
                                                            int total_tiles) {
    __shared__ Tap tys[kResRows];
    for (int gt = blockIdx.x; gt < total_tiles; gt += gridDim.x) {
        int lo = 0, hi = njobs - 1;  // last job with tile_base <= gt
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (jobs[mid].tile_base <= gt)
                lo = mid;
            else
                hi = mid - 1;
        }
        const ResampleJob& J = jobs[lo];
        const int tile = gt - J.tile_base;
        const int tcols = (J.dw + kResCols - 1) / kResCols;
        const int ty = tile / tcols, tx = tile - ty * tcols;
        const int ybase = ty * kResRows, x = tx * kResCols + threadIdx.x;
        __syncthreads();
        if (threadIdx.x < kResRows && ybase + threadIdx.x < J.dh)
            tys[threadIdx.x] = make_tap_s(ybase + threadIdx.x, J.sh, J.sy);
        __syncthreads();
        if (J.idx32) {
            switch (J.nplanes) {
                case 1: resample_tile<1, int>(J, x, ybase, tys); break;
                case 3: resample_tile<3, int>(J, x, ybase, tys); break;
                case 6: resample_tile<6, int>(J, x, ybase, tys); break;
                default: resample_tile_generic(J, x, ybase, tys); break;
            }
        } else {
            switch (J.nplanes) {
                case 1: resample_tile<1, long long>(J, x, ybase, tys); break;
                case 3: resample_tile<3, long long>(J, x, ybase, tys); break;
                case 6: resample_tile<6, long long>(J, x, ybase, tys); break;
                default: resample_tile_generic(J, x, ybase, tys); break;
            }
        }
    }
}

// ----------------------------------------------------------------------------
// Upsampling of the six F/B planes from the previous level, for scales
// sw/dw, sh/dh <= kUpMaxScale (level sizes grow by ~2x; larger scales take the
// generic resample kernel).  A tile of 8 x 128 outputs reads at most
// kUpSR x kUpSC source texels per plane.  Each block double-buffers the
// staged windows of two consecutive tiles in shared memory (cp.async), so the
// next tile's loads overlap this tile's interpolation; every output takes its
// four taps from shared memory with compile-time plane offsets.  Same
// arithmetic as resample_tile (bitwise identical results).
#ifndef FGM_UP_ROWS
#define FGM_UP_ROWS 8
#endif
#ifndef FGM_UP_THREADS
#define FGM_UP_THREADS 128
#endif
constexpr int kUpCols = 128, kUpRows = FGM_UP_ROWS, kUpThreads = FGM_UP_THREADS, kUpWarps = kUpThreads / 32;
static_assert(kUpRows % kUpWarps == 0, "every warp takes the same number of tile rows");
constexpr double kUpMaxScale = 0.625;
constexpr int kUpSR = (kUpRows - 1) * 5 / 8 + 4;  // >= ceil((rows-1) * 0.625) + 3
// window columns: ceil(127 * 0.625) + 3 = 83, plus up to 3 + 3 for the
// 16-byte block alignment of both ends, rounded to 16 bytes
constexpr int kUpSC = 92;
constexpr int kUpPlane = kUpSR * kUpSC;
constexpr int kUpBuf = 6 * kUpPlane;

__device__ __forceinline__ void cp_async_f32(unsigned sdst, const float* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_v4(unsigned sdst, const float* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void st_cs(float* p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

struct UpTile {
    int job, y0, x0, nrows, ncols, r0, c0, nr, nc;  // nr x nc: staged source window from (r0, c0)
};

// Tile geometry and source window; `job` advances monotonically per block.
// With 16-byte staging (v4) the window starts at the 4-aligned column below
// the first tap.
__device__ __forceinline__ UpTile up_tile(const ResampleJob* __restrict__ jobs, int njobs, int gt, int job) {
    while (job + 1 < njobs && jobs[job + 1].tile_base <= gt) ++job;
    const ResampleJob& J = jobs[job];
    const int tile = gt - J.tile_base;
    const int tcols = (J.dw + kUpCols - 1) / kUpCols;
    const int tyi = tile / tcols, txi = tile - tyi * tcols;
    UpTile t;
    t.job = job;
    t.y0 = tyi * kUpRows;
    t.x0 = txi * kUpCols;
    t.nrows = min(kUpRows, J.dh - t.y0);
    t.ncols = min(kUpCols, J.dw - t.x0);
    t.r0 = make_tap_s(t.y0, J.sh, J.sy).i0;
    const int c0 = make_tap_s(t.x0, J.sw, J.sx).i0;
    // exact window: up to the last row's / column's i1
    t.nr = make_tap_s(t.y0 + t.nrows - 1, J.sh, J.sy).i1 - t.r0 + 1;
    const int c1 = make_tap_s(t.x0 + t.ncols - 1, J.sw, J.sx).i1;
    const bool v4 = ((reinterpret_cast<uintptr_t>(J.src) | uintptr_t(J.spitch) | uintptr_t(J.spstride)) & 3) == 0 &&
                    (reinterpret_cast<uintptr_t>(J.src) & 15) == 0;
    t.c0 = v4 ? (c0 & ~3) : c0;
    t.nc = v4 ? -(((c1 | 3) - t.c0 + 1) >> 2) : c1 - c0 + 1;  // < 0: number of 16-byte blocks
    return t;
}

// Issue the cp.async loads of a tile's window and its row taps (threads
// 0..7) into buffer b.  16-byte blocks when the source rows allow it (level
// buffers are pitched to 4 floats; the blocks may read into the row padding,
// which no tap uses).
__device__ __forceinline__ void up_stage(const ResampleJob& J, const UpTile& t, unsigned sbuf, Tap* tys, int tid) {
    const int nr = t.nr;  // <= kUpSR at scales <= kUpMaxScale
    const int sp = J.spitch;
    const long long sps = J.spstride;
    const int warp = tid >> 5, lane = tid & 31;
    if (t.nc < 0) {
        const int nb = -t.nc;  // blocks per row (<= kUpSC / 4 = 23 < 32: one per lane)
#pragma unroll
        for (int p = 0; p < 6; ++p) {
            const float* sp0 = J.src + p * sps + (long long)t.r0 * sp + t.c0 + 4 * lane;
            const unsigned d0 = sbuf + 4u * unsigned(p * kUpPlane + 4 * lane);
            if (lane < nb)
                for (int r = warp; r < nr; r += kUpThreads / 32)
                    cp_async_v4(d0 + 4u * unsigned(r * kUpSC), sp0 + (long long)r * sp);
        }
    } else {
        const int nc = t.nc;
#pragma unroll
        for (int p = 0; p < 6; ++p) {
            const float* sp0 = J.src + p * sps + (long long)t.r0 * sp + t.c0;
            for (int r = warp; r < nr; r += kUpThreads / 32) {
                const float* srow = sp0 + (long long)r * sp;
                const unsigned drow = sbuf + 4u * unsigned(p * kUpPlane + r * kUpSC);
                for (int c = lane; c < nc; c += 32) cp_async_f32(drow + 4u * c, srow + c);
            }
        }
    }
    if (tid < t.nrows) tys[tid] = make_tap_s(t.y0 + tid, J.sh, J.sy);
}

__global__ void __launch_bounds__(kUpThreads) upsample_kernel(const ResampleJob* __restrict__ jobs, int njobs,
                                                              int total_tiles) {
    extern __shared__ float4 up_sm4[];
    float* sm = reinterpret_cast<float*>(up_sm4);
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    __shared__ Tap tys[2][kUpRows];
    const int tid = threadIdx.x;
    int gt = blockIdx.x;
    if (gt >= total_tiles) return;
    UpTile cur = up_tile(jobs, njobs, gt, 0);
    up_stage(jobs[cur.job], cur, sbase, tys[0], tid);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int it = 0;; ++it) {
        const int b = it & 1;
        const int gn = gt + gridDim.x;
        UpTile nxt = cur;
        if (gn < total_tiles) {  // stage the next tile into the other buffer
            nxt = up_tile(jobs, njobs, gn, cur.job);
            up_stage(jobs[nxt.job], nxt, sbase + 4u * unsigned((b ^ 1) * kUpBuf), tys[b ^ 1], tid);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
        __syncthreads();  // this tile's window and taps are visible
        {
            // thread = (lane l, warp rp): columns x0 + l + 32i (i < 4), rows
            // rp, rp + 4, ...  Lanes read neighbouring (or equal) staged words:
            // no bank conflicts; stores are 128-byte warp rows.  Columns past
            // the tile's end are computed on a clamped column and not stored.
            const ResampleJob& J = jobs[cur.job];
            const int l = tid & 31, rp = tid >> 5;
            int ca[4], cb[4];
            float tx[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const Tap t = make_tap_s(min(cur.x0 + l + 32 * i, J.dw - 1), J.sw, J.sx);
                ca[i] = t.i0 - cur.c0;
                cb[i] = t.i1 - cur.c0;
                tx[i] = t.t;
            }
            const float* buf = sm + b * kUpBuf;
            const long long dps = J.dpstride;
            float* dcol = J.dst + cur.x0 + l;
#pragma unroll
            for (int h = 0; h < kUpRows / kUpWarps; ++h) {
                const int rr = rp + kUpWarps * h;  // warp-uniform
                if (rr >= cur.nrows) break;
                const Tap ty = tys[b][rr];
                const float* ra = buf + (ty.i0 - cur.r0) * kUpSC;
                const float* rc = buf + (ty.i1 - cur.r0) * kUpSC;
                float* d = dcol + (long long)(cur.y0 + rr) * J.dpitch;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (l + 32 * i >= cur.ncols) break;  // (the tile's last column block only)
                    const float* a0 = ra + ca[i];
                    const float* a1 = ra + cb[i];
                    const float* c0 = rc + ca[i];
                    const float* c1 = rc + cb[i];
                    float v[6];
#pragma unroll
                    for (int p = 0; p < 6; p += 2) {  // plane pairs: packed fp32x2 arithmetic
                        const int o = p * kUpPlane, q = o + kUpPlane;
                        const float2 r = bilerp2(make_float2(a0[o], a0[q]), make_float2(a1[o], a1[q]),
                                                 make_float2(c0[o], c0[q]), make_float2(c1[o], c1[q]), tx[i], ty.t);
                        v[p] = r.x;
                        v[p + 1] = r.y;
                    }
                    // streaming stores: the next level's sweep reads them once, much later
#pragma unroll
                    for (int p = 0; p < 6; ++p) st_cs(d + p * dps + 32 * i, v[p]);
                }
            }
        }
        __syncthreads();  // buffer b is free for the tile after next
        if (gn >= total_tiles) break;
        gt = gn;
        cur = nxt;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

int upsample_tiles(int dw, int dh) { return ((dw + kUpCols - 1) / kUpCols) * ((dh + kUpRows - 1) / kUpRows); }

cudaError_t launch_upsample(const ResampleJob* jobs_dev, int njobs, long long total_tiles, cudaStream_t s) {
    if (njobs <= 0 || total_tiles <= 0) return cudaSuccess;
    constexpr size_t smem = size_t(2) * kUpBuf * sizeof(float);
    static PerDevice<int2> cfg;  // (SMs, blocks per SM)
    int2 c;
    cudaError_t e = cfg.get(c, [&](int dev, int2& v) {
        cudaError_t r = cudaFuncSetAttribute(upsample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (r == cudaSuccess) r = cudaDeviceGetAttribute(&v.x, cudaDevAttrMultiProcessorCount, dev);
        if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v.y, upsample_kernel, kUpThreads, smem);
        v.y = std::max(v.y, 1);
        return r;
    });
    if (e != cudaSuccess) return e;
    const int gx = int(std::min<long long>(total_tiles, (long long)c.x * c.y));
    upsample_kernel<<<gx, kUpThreads, smem, s>>>(jobs_dev, njobs, int(total_tiles));
    return cudaGetLastError();
}

bool upsample_ok(int sw, int sh, int dw, int dh) {
    return !(sw == dw && sh == dh) && double(sw) / double(dw) <= kUpMaxScale &&
           double(sh) / double(dh) <= kUpMaxScale;
}

int resample_tiles(int dw, int dh) { return ((dw + kResCols - 1) / kResCols) * ((dh + kResRows - 1) / kResRows); }

cudaError_t launch_resample(const ResampleJob* jobs_dev, int njobs, long long total_tiles, cudaStream_t s,
                            int blocks_per_sm) {
    if (njobs <= 0 || total_tiles <= 0) return cudaSuccess;
    static PerDevice<int> cfg;  // SMs
    int sms = 0;
    cudaError_t e = cfg.get(sms, [](int dev, int& v) { return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev); });
    if (e != cudaSuccess) return e;
    // blocks_per_sm 0: one tile per block (no persistent blocks holding SM slots)
    const int gx = int(blocks_per_sm > 0 ? std::min<long long>(total_tiles, (long long)sms * blocks_per_sm) : total_tiles);
    resample_kernel<<<gx, kResCols, 0, s>>>(jobs_dev, njobs, int(total_tiles));
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// K1': the I/alpha pyramid in one pass.  Every sub-top level is a bilinear
// resize of the FULL-RESOLUTION input (multilevel.cpp:154-156 resizes the
// original for each level), so the per-level K1 launches read the input ~2x
// over (all rows for the ~2x level, half of them for the ~4x level, ...).
// Here a block stages a kPyrTH x kPyrTW full-res tile (plus one overlap row
// and column) of the four planes in shared memory once and emits, for every
// level, the outputs whose first taps (i0) fall inside the tile: their second
// taps (i1 = i0 + 1 or the clamped edge) are then inside the staged window.
// Taps and arithmetic are those of resample_tile (bitwise identical output).
constexpr int kPyrThreads = 256;
constexpr int kPyrSW = kPyrTW + 4;           // staged row: 33 16-byte chunks (column 128 + padding)
constexpr int kPyrPlane = (kPyrTH + 1) * kPyrSW;
constexpr int kPyrBuf = 4 * kPyrPlane;

// Smallest destination index whose first tap is >= r (dst if none): the
// analytic estimate, then exact checks with the reference taps (i0 is
// non-decreasing in the destination index).
__device__ __forceinline__ int pyr_first(int r, int src, int dst, double scale, double rscale) {
    if (r <= 0) return 0;
    if (r > src - 1) return dst;
    int d = int(ceil((double(r) + 0.5) * rscale - 0.5));  // (an estimate: the loops below are exact)
    d = max(0, min(d, dst));
    while (d > 0 && make_tap_s(d - 1, src, scale).i0 >= r) --d;
    while (d < dst && make_tap_s(d, src, scale).i0 < r) ++d;
    return d;
}

struct PyrTile {
    int job, R0, C0, rows, cols;
};

// `job` advances monotonically per block (tiles are walked in increasing order)
__device__ __forceinline__ PyrTile pyr_tile(const PyrJob* __restrict__ jobs, int njobs, int gt, int job) {
    int lo = job;
    while (lo + 1 < njobs && jobs[lo + 1].tile_base <= gt) ++lo;
    const PyrJob& J = jobs[lo];
    const int tile = gt - J.tile_base;
    const int tyi = tile / J.tcols, txi = tile - tyi * J.tcols;
    PyrTile t;
    t.job = lo;
    t.R0 = tyi * kPyrTH;
    t.C0 = txi * kPyrTW;
    t.rows = min(kPyrTH + 1, J.H - t.R0);
    t.cols = min(kPyrTW + 1, J.W - t.C0);
    return t;
}

// cp.async staging of a tile's four planes (16-byte chunks when every row of
// the input is 16-byte aligned; the chunk past the row end is zero-filled and
// never read), and the per-level output ranges of the tile (threads < 4 nlev).
__device__ __forceinline__ void pyr_stage(const PyrJob& J, const PyrTile& t, unsigned sbuf, int (*rng)[4], int tid) {
    const int W = J.W;
    const long long HW = (long long)W * J.H;
    const bool v4 = (W & 3) == 0 && ((reinterpret_cast<uintptr_t>(J.img) | reinterpret_cast<uintptr_t>(J.alpha)) & 15) == 0;
    const int warp = tid >> 5, lane = tid & 31;
    const float* img = J.img + (long long)t.R0 * W + t.C0;
    const float* alp = J.alpha + (long long)t.R0 * W + t.C0;
    if (v4) {
        const int nch = (t.cols + 3) >> 2;  // <= 33 chunks per row
        for (int r = warp; r < t.rows; r += kPyrThreads / 32) {
            for (int c4 = lane; c4 < nch; c4 += 32) {
                const int c = 4 * c4;
                const int bytes = min(4, W - (t.C0 + c)) * 4;
                const long long g = (long long)r * W + c;
                const unsigned d = sbuf + 4u * unsigned(r * kPyrSW + c);
                const float* src[4] = {img + g, img + HW + g, img + 2 * HW + g, alp + g};
#pragma unroll
                for (int p = 0; p < 4; ++p)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d + 4u * unsigned(p * kPyrPlane)),
                                 "l"(src[p]), "r"(bytes)
                                 : "memory");
            }
        }
    } else {
        for (int r = warp; r < t.rows; r += kPyrThreads / 32) {
            for (int c = lane; c < t.cols; c += 32) {
                const long long g = (long long)r * W + c;
                const unsigned d = sbuf + 4u * unsigned(r * kPyrSW + c);
                const float* src[4] = {img + g, img + HW + g, img + 2 * HW + g, alp + g};
#pragma unroll
                for (int p = 0; p < 4; ++p) cp_async_f32(d + 4u * unsigned(p * kPyrPlane), src[p]);
            }
        }
    }
    if (tid < 4 * J.nlev) {
        const int l = tid >> 2, b = tid & 3;
        rng[l][b] = b < 2 ? pyr_first(t.R0 + (b & 1) * kPyrTH, J.H, J.lh[l], J.sy[l], J.rsy[l])
                          : pyr_first(t.C0 + (b & 1) * kPyrTW, W, J.lw[l], J.sx[l], J.rsx[l]);
    }
}

// Persistent blocks, double-buffered: the next tile's loads are in flight
// while this tile's outputs are interpolated.
__global__ void __launch_bounds__(kPyrThreads) pyramid_kernel(const PyrJob* __restrict__ jobs, int njobs,
                                                              int total_tiles) {
    extern __shared__ float4 pyr_sm4[];
    float* sm = reinterpret_cast<float*>(pyr_sm4);
    const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(sm));
    __shared__ int rng[2][kMaxPyr][4];  // per buffer and level: first/end output row, first/end output column
    const int tid = threadIdx.x;
    int gt = blockIdx.x;
    if (gt >= total_tiles) return;
    PyrTile cur = pyr_tile(jobs, njobs, gt, 0);
    pyr_stage(jobs[cur.job], cur, sbase, rng[0], tid);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int it = 0;; ++it) {
        const int b = it & 1;
        const int gn = gt + gridDim.x;
        PyrTile nxt = cur;
        if (gn < total_tiles) {
            nxt = pyr_tile(jobs, njobs, gn, cur.job);
            pyr_stage(jobs[nxt.job], nxt, sbase + 4u * unsigned((b ^ 1) * kPyrBuf), rng[b ^ 1], tid);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 1;" ::: "memory");
        __syncthreads();  // this tile's window and ranges are visible
        {
            // warps over output rows, lanes over output columns (coalesced
            // stores, no index division); a lane's x-taps are computed once per
            // level and reused for every row
            const PyrJob& J = jobs[cur.job];
            const int W = J.W, H = J.H, nlev = J.nlev;
            const int warp = tid >> 5, lane = tid & 31;
            const float* buf = sm + b * kPyrBuf;
            for (int l = 0; l < nlev; ++l) {
                const int dy0 = rng[b][l][0], ny = rng[b][l][1] - dy0, dx0 = rng[b][l][2], nx = rng[b][l][3] - dx0;
                if (ny <= 0 || nx <= 0) continue;
                const int pitch = J.pitch[l];
                const long long ps = (long long)pitch * J.lh[l];
                float* out = J.out[l] + (long long)dy0 * pitch + dx0;
                const double sx = J.sx[l], sy = J.sy[l];
                for (int x0 = 0; x0 < nx; x0 += 32) {
                    const int xi = x0 + lane;
                    if (xi >= nx) break;
                    const Tap tx = make_tap_s(dx0 + xi, W, sx);
                    const int cx = tx.i0 - cur.C0, dx = tx.i1 - tx.i0;
                    for (int yi = warp; yi < ny; yi += kPyrThreads / 32) {
                        const Tap ty = make_tap_s(dy0 + yi, H, sy);
                        const int a0 = (ty.i0 - cur.R0) * kPyrSW + cx;
                        const int c0 = (ty.i1 - cur.R0) * kPyrSW + cx;
                        float* d = out + (long long)yi * pitch + xi;
                        float v[4];
#pragma unroll
                        for (int p = 0; p < 4; ++p) {
                            const float* s = buf + p * kPyrPlane;
                            v[p] = bilerp(s[a0], s[a0 + dx], s[c0], s[c0 + dx], tx.t, ty.t);
                        }
#pragma unroll
                        for (int p = 0; p < 4; ++p) d[p * ps] = v[p];
                    }
                }
            }
        }
        __syncthreads();  // buffer b (and its ranges) are free for the tile after next
        if (gn >= total_tiles) break;
        gt = gn;
        cur = nxt;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

cudaError_t launch_pyramid(const PyrJob* jobs_dev, int njobs, long long total_tiles, cudaStream_t s) {
    if (njobs <= 0 || total_tiles <= 0) return cudaSuccess;
    constexpr size_t smem = size_t(2) * kPyrBuf * sizeof(float);
    static PerDevice<int2> cfg;  // (SMs, blocks per SM)
    int2 c;
    cudaError_t e = cfg.get(c, [&](int dev, int2& v) {
        cudaError_t r = cudaFuncSetAttribute(pyramid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (r == cudaSuccess) r = cudaDeviceGetAttribute(&v.x, cudaDevAttrMultiProcessorCount, dev);
        if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v.y, pyramid_kernel, kPyrThreads, smem);
        v.y = std::max(v.y, 1);
        return r;
    });
    if (e != cudaSuccess) return e;
    const int gx = int(std::min<long long>(total_tiles, (long long)c.x * c.y));
    pyramid_kernel<<<gx, kPyrThreads, smem, s>>>(jobs_dev, njobs, int(total_tiles));
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// K5 layout kernels of the HWC boundary (python/bindings.cpp:20-53): an
// interleaved (h, w, ch) image of T (float or double) to planar fp32 with the
// binding's clamp01 on every input value, and planar fp32 back to (h, w, 3).
template <typename T>
__global__ void hwc_to_planar_kernel(const T* __restrict__ src, long long n, int ch, float* __restrict__ dst) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
        for (int c = 0; c < ch; ++c) {
            const double v = double(src[i * ch + c]);
            dst[(long long)c * n + i] = float(v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v));  // clamp01 in the source type
        }
}

template <typename T>
__global__ void planar_to_hwc_kernel(const float* __restrict__ src, long long n, int ch, T* __restrict__ dst) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
        for (int c = 0; c < ch; ++c) dst[i * ch + c] = T(src[(long long)c * n + i]);
}

cudaError_t launch_hwc_to_planar(const void* src, bool f64, long long n, int ch, float* dst, cudaStream_t s) {
    const int gx = std::max(1, int(std::min<long long>((n + 255) / 256, 148 * 16)));
    if (f64)
        hwc_to_planar_kernel<double><<<gx, 256, 0, s>>>(static_cast<const double*>(src), n, ch, dst);
    else
        hwc_to_planar_kernel<float><<<gx, 256, 0, s>>>(static_cast<const float*>(src), n, ch, dst);
    return cudaGetLastError();
}

cudaError_t launch_planar_to_hwc(const float* src, long long n, int ch, void* dst, bool f64, cudaStream_t s) {
    const int gx = std::max(1, int(std::min<long long>((n + 255) / 256, 148 * 16)));
    if (f64)
        planar_to_hwc_kernel<double><<<gx, 256, 0, s>>>(src, n, ch, static_cast<double*>(dst));
    else
        planar_to_hwc_kernel<float><<<gx, 256, 0, s>>>(src, n, ch, static_cast<float*>(dst));
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// Quality metrics (metrics.cpp:75-145): alpha-weighted SAD, "MSE" (a weighted
// sum) and the Gaussian-derivative gradient error over the translucent region
// 0 < alpha < 1, in fp64 with the reference's per-pixel operation order (no
// FMA contraction: __dmul_rn/__dadd_rn), one partial sum per block (summed on
// the host in block order: deterministic).
constexpr int kMetThreads = 256;

__device__ __forceinline__ double conv_at(const float* p, int x, int y, int w, int h, bool along_x,
                                          const double* kern, int r) {
    double acc = 0.0;  // convolve_axis, metrics.cpp:35-57
    for (int k = -r; k <= r; ++k) {
        int xx = x, yy = y;
        if (along_x) {
            xx = x + k;
            xx = xx < 0 ? 0 : (xx > w - 1 ? w - 1 : xx);
        } else {
            yy = y + k;
            yy = yy < 0 ? 0 : (yy > h - 1 ? h - 1 : yy);
        }
        acc = __dadd_rn(acc, __dmul_rn(kern[k + r], double(p[(long long)yy * w + xx])));
    }
    return acc;
}

__global__ void __launch_bounds__(kMetThreads) metrics_kernel(const float* __restrict__ est,
                                                              const float* __restrict__ gt,
                                                              const float* __restrict__ alpha, int w, int h, int nch,
                                                              const double* __restrict__ kern, int r,
                                                              double* __restrict__ partial) {
    const long long n = (long long)w * h;
    double s_sad = 0.0, s_mse = 0.0, s_grad = 0.0, s_cnt = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = double(alpha[i]);
        if (!(a > 0.0 && a < 1.0)) continue;
        const int x = int(i % w), y = int(i / w);
        double d_abs = 0.0, d_sq = 0.0;
        for (int c = 0; c < nch; ++c) {
            const double e = __dadd_rn(double(est[c * n + i]), -double(gt[c * n + i]));
            d_abs = __dadd_rn(d_abs, fabs(e));
            d_sq = __dadd_rn(d_sq, __dmul_rn(e, e));
        }
        s_sad = __dadd_rn(s_sad, __dmul_rn(a, d_abs));
        s_mse = __dadd_rn(s_mse, __dmul_rn(a, d_sq));
        for (int c = 0; c < nch; ++c) {
            const float* pe = est + c * n;
            const float* pg = gt + c * n;
            const double gx = __dadd_rn(conv_at(pe, x, y, w, h, true, kern, r), -conv_at(pg, x, y, w, h, true, kern, r));
            const double gy =
                __dadd_rn(conv_at(pe, x, y, w, h, false, kern, r), -conv_at(pg, x, y, w, h, false, kern, r));
            s_grad = __dadd_rn(s_grad, __dmul_rn(a, __dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy))));
        }
        s_cnt += 1.0;
    }
    __shared__ double red[4][kMetThreads];
    red[0][threadIdx.x] = s_sad;
    red[1][threadIdx.x] = s_mse;
    red[2][threadIdx.x] = s_grad;
    red[3][threadIdx.x] = s_cnt;
    __syncthreads();
    for (int o = kMetThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 4) partial[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}

int metrics_blocks(long long n) { return int(std::max<long long>(1, std::min<long long>((n + kMetThreads - 1) / kMetThreads, 148 * 8))); }

cudaError_t launch_metrics(const float* est, const float* gt, const float* alpha, int w, int h, int nch,
                           const double* kern, int r, double* partial, int blocks, cudaStream_t s) {
    metrics_kernel<<<blocks, kMetThreads, 0, s>>>(est, gt, alpha, w, h, nch, kern, r, partial);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------
// Compose epilogue (image.cpp:39-57): out = clamp01(a * f + (1 - a) * b) per
// plane, in the reference's operation order (a*f, (1-a)*b, add; no FMA).
__global__ void compose_kernel(const float* __restrict__ fg, const float* __restrict__ bg,
                               const float* __restrict__ alpha, long long n, int nch, float* out) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float a = alpha[i], ia = __fsub_rn(1.0f, a);
        for (int c = 0; c < nch; ++c) {
            const long long j = (long long)c * n + i;
            out[j] = __saturatef(__fadd_rn(__fmul_rn(a, fg[j]), __fmul_rn(ia, bg[j])));
        }
    }
}

cudaError_t launch_compose(const float* fg, const float* bg, const float* alpha, long long n, int nch, float* out,
                           cudaStream_t s) {
    const int gx = int(std::min<long long>((n + 255) / 256, 148 * 16));
    compose_kernel<<<std::max(gx, 1), 256, 0, s>>>(fg, bg, alpha, n, nch, out);
    return cudaGetLastError();
}

// ============================================================================
// K4: coarse levels, in fp64 with the reference's own operation order, so the
// coarse prefix of every solve is bitwise the reference's (given the same
// inputs).  One CTA per image.  Per level: I/alpha resampled from the
// full-resolution input (global; fp64 when the caller passed fp64, else the
// fp32 input upcast exactly), F/B from the previous level (shared), then
// `iterations` sweeps in place in shared memory along the wavefront
// t = x + y + 2k: pixel (x,y) of sweep k reads only values of step t-1 or
// earlier, and pixels updated in one step never read each other (equal x + y
// parity) -- the same values the sequential scanline sweep reads
// (multilevel.cpp:91-120).  No FMA contraction anywhere (__d*_rn): the
// reference is built with -ffp-contract=off (CMakeLists.txt:23-24).
// ============================================================================
constexpr int kCoarseThreads = 256;

// I (3) + alpha + two F/B buffers (6 each), fp64
size_t coarse_smem_bytes() { return size_t(16) * kCoarseCap * sizeof(double); }

__device__ __forceinline__ double dclamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

// image.cpp:98-102: top = a + t (b - a), bot = c + t (d - c), clamp01(top + ty (bot - top))
__device__ __forceinline__ double dbilerp(double a, double b, double c, double d, double tx, double ty) {
    const double top = __dadd_rn(a, __dmul_rn(tx, __dsub_rn(b, a)));
    const double bot = __dadd_rn(c, __dmul_rn(tx, __dsub_rn(d, c)));
    return dclamp01(__dadd_rn(top, __dmul_rn(ty, __dsub_rn(bot, top))));
}

// make_taps (image.cpp:71-83) with t kept in fp64
struct Tap64 {
    int i0, i1;
    double t;
};
__device__ __forceinline__ Tap64 make_tap64(int d, int src, double scale) {
    double f = __dadd_rn(__dmul_rn(__dadd_rn(double(d), 0.5), scale), -0.5);
    if (f < 0.0) f = 0.0;
    const double max_f = double(src - 1);
    if (f > max_f) f = max_f;
    const int i0 = int(f);
    return {i0, min(i0 + 1, src - 1), __dsub_rn(f, double(i0))};
}

// One pixel of sweep (multilevel.cpp:93-118), PixelSystem's order
// (multilevel.hpp:45-75): init, the four clamped neighbours L, R, U, D, the
// adjugate solve with inv_det = 1 / det, clamp01.
__device__ __forceinline__ void coarse_update(const double* __restrict__ sI, const double* __restrict__ sA,
                                              double* __restrict__ fb, int x, int y, int w, int h, double eps,
                                              double omega) {
    const int n = w * h;
    const int i = y * w + x;
    const int jn[4] = {x > 0 ? i - 1 : i, x < w - 1 ? i + 1 : i, y > 0 ? i - w : i, y < h - 1 ? i + w : i};
    const double ai = sA[i];
    const double u0 = ai, u1 = __dsub_rn(1.0, ai);
    double diag0 = __dmul_rn(u0, u0), diag1 = __dmul_rn(u1, u1);
    const double off = __dmul_rn(u0, u1);
    double rf[3], rb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double Ic = sI[c * n + i];
        rf[c] = __dmul_rn(Ic, u0);
        rb[c] = __dmul_rn(Ic, u1);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int j = jn[t];
        const double dalpha = __dadd_rn(eps, __dmul_rn(omega, fabs(__dsub_rn(ai, sA[j]))));
        diag0 = __dadd_rn(diag0, dalpha);
        diag1 = __dadd_rn(diag1, dalpha);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            rf[c] = __dadd_rn(rf[c], __dmul_rn(dalpha, fb[c * n + j]));
            rb[c] = __dadd_rn(rb[c], __dmul_rn(dalpha, fb[(3 + c) * n + j]));
        }
    }
    const double inv_det = __ddiv_rn(1.0, __dsub_rn(__dmul_rn(diag0, diag1), __dmul_rn(off, off)));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        fb[c * n + i] = dclamp01(__dmul_rn(__dsub_rn(__dmul_rn(diag1, rf[c]), __dmul_rn(off, rb[c])), inv_det));
        fb[(3 + c) * n + i] = dclamp01(__dmul_rn(__dsub_rn(__dmul_rn(diag0, rb[c]), __dmul_rn(off, rf[c])), inv_det));
    }
}

// the full-resolution input value of plane c (3 = alpha) at index k
__device__ __forceinline__ double full_res(const CoarseJob& J, int c, long long k, long long fps) {
    if (J.img64) return c < 3 ? J.img64[c * fps + k] : J.alpha64[k];
    return double(c < 3 ? __ldg(J.img + c * fps + k) : __ldg(J.alpha + k));
}

__global__ void __launch_bounds__(kCoarseThreads) coarse_kernel(const CoarseJob* __restrict__ jobs, double eps,
                                                                 double omega) {
    extern __shared__ double smd[];
    const CoarseJob& J = jobs[blockIdx.x];
    const int cap = kCoarseCap;
    double* sI = smd;
    double* sA = smd + 3 * cap;
    double* sFB[2] = {smd + 4 * cap, smd + 10 * cap};
    const int W = J.W, H = J.H;
    const long long fps = (long long)W * H;
    int pw = 1, ph = 1;
    const int nlev = J.nlev;
    for (int l = 0; l < nlev; ++l) {
        const int w = J.lw[l], h = J.lh[l], K = J.lit[l];
        const int n = w * h, pn = pw * ph;
        double* cur = sFB[l & 1];
        const double* prv = sFB[(l & 1) ^ 1];
        const bool ident = (w == W && h == H);
        const bool same = (w == pw && h == ph);
        const double sxf = __ddiv_rn(double(W), double(w)), syf = __ddiv_rn(double(H), double(h));
        const double sxp = __ddiv_rn(double(pw), double(w)), syp = __ddiv_rn(double(ph), double(h));
        for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
            const int y = idx / w, x = idx - y * w;
            if (ident) {  // the last level resamples the original: identity copy (image.cpp:116,127)
#pragma unroll
                for (int c = 0; c < 3; ++c) sI[c * n + idx] = full_res(J, c, idx, fps);
                sA[idx] = full_res(J, 3, idx, fps);
            } else {
                const Tap64 tx = make_tap64(x, W, sxf), ty = make_tap64(y, H, syf);
                const long long r0 = (long long)ty.i0 * W, r1 = (long long)ty.i1 * W;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const double v = dbilerp(full_res(J, c, r0 + tx.i0, fps), full_res(J, c, r0 + tx.i1, fps),
                                             full_res(J, c, r1 + tx.i0, fps), full_res(J, c, r1 + tx.i1, fps), tx.t,
                                             ty.t);
                    if (c < 3)
                        sI[c * n + idx] = v;
                    else
                        sA[idx] = v;
                }
            }
            if (l == 0) {  // F, B start as 1x1 zeros (multilevel.cpp:155-156)
#pragma unroll
                for (int p = 0; p < 6; ++p) cur[p * n + idx] = 0.0;
            } else if (same) {
#pragma unroll
                for (int p = 0; p < 6; ++p) cur[p * n + idx] = prv[p * pn + idx];
            } else {
                const Tap64 tx = make_tap64(x, pw, sxp), ty = make_tap64(y, ph, syp);
                const int r0 = ty.i0 * pw, r1 = ty.i1 * pw;
#pragma unroll
                for (int p = 0; p < 6; ++p) {
                    const double* s = prv + p * pn;
                    cur[p * n + idx] = dbilerp(s[r0 + tx.i0], s[r0 + tx.i1], s[r1 + tx.i0], s[r1 + tx.i1], tx.t, ty.t);
                }
            }
        }
        __syncthreads();
        const int T = (w - 1) + (h - 1) + 2 * (K - 1) + 1;
        const int items = h * K;
        for (int t = 0; t < T; ++t) {
            for (int it = threadIdx.x; it < items; it += blockDim.x) {
                const int k = it / h, y = it - k * h;
                const int x = t - y - 2 * k;
                if (x >= 0 && x < w) coarse_update(sI, sA, cur, x, y, w, h, eps, omega);
            }
            __syncthreads();
        }
        if (J.lvl_fg[l]) {
            for (int idx = threadIdx.x; idx < 3 * n; idx += blockDim.x) {
                J.lvl_fg[l][idx] = float(cur[idx]);
                J.lvl_bg[l][idx] = float(cur[3 * n + idx]);
            }
        }
        pw = w;
        ph = h;
    }
    const double* fin = sFB[(nlev - 1) & 1];
    const int n = pw * ph;
    for (int idx = threadIdx.x; idx < 3 * n; idx += blockDim.x) {
        const int c = idx / n, i = idx - c * n, y = i / pw, x = i - y * pw;
        const long long o = c * J.out_pstride + (long long)y * J.out_pitch + x;
        J.fg_out[o] = float(fin[idx]);
        J.bg_out[o] = float(fin[3 * n + idx]);
        if (J.fg_out64) {  // fp64 host path, image entirely coarse: the exact values
            J.fg_out64[o] = fin[idx];
            J.bg_out64[o] = fin[3 * n + idx];
        }
    }
}

cudaError_t launch_coarse(const CoarseJob* jobs_dev, int njobs, double eps, double omega, cudaStream_t s) {
    if (njobs <= 0) return cudaSuccess;
    static PerDevice<int> attr;  // the > 48 KB shared-memory opt-in, per device
    int unused = 0;
    cudaError_t e = attr.get(unused, [](int, int&) {
        return cudaFuncSetAttribute(coarse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(coarse_smem_bytes()));
    });
    if (e != cudaSuccess) return e;
    coarse_kernel<<<njobs, kCoarseThreads, coarse_smem_bytes(), s>>>(jobs_dev, eps, omega);
    return cudaGetLastError();
}

// ============================================================================
// K5: fp64 <-> fp32 planar conversion for the C++ drop-in boundary.
// ============================================================================
__global__ void f64_to_f32_kernel(const double* __restrict__ s, float* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        d[i] = float(s[i]);
}
__global__ void f32_to_f64_kernel(const float* __restrict__ s, double* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        d[i] = double(s[i]);
}
cudaError_t launch_f64_to_f32(const double* src, float* dst, size_t n, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const int g = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    f64_to_f32_kernel<<<g, 256, 0, s>>>(src, dst, n);
    return cudaGetLastError();
}
cudaError_t launch_f32_to_f64(const float* src, double* dst, size_t n, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const int g = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    f32_to_f64_kernel<<<g, 256, 0, s>>>(src, dst, n);
    return cudaGetLastError();
}

}  // namespace fgm
