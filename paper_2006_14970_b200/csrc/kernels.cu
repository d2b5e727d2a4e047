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

template <int NP>
__device__ __forceinline__ void resample_tile(const ResampleJob& J, int x, int ybase, const Tap* tys) {
    if (x >= J.dw) return;
    const int yend = min(kResRows, J.dh - ybase);
    if (J.sw == J.dw && J.sh == J.dh) {  // resize to the same size: unclamped copy
        for (int r = 0; r < yend; ++r) {
            const long long is = (long long)(ybase + r) * J.spitch + x, id = (long long)(ybase + r) * J.dpitch + x;
            float v[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) v[p] = __ldg(J.src + p * J.spstride + is);
#pragma unroll
            for (int p = 0; p < NP; ++p) J.dst[p * J.dpstride + id] = v[p];
        }
        return;
    }
    const Tap tx = make_tap_s(x, J.sw, J.sx);
    for (int r = 0; r < yend; ++r) {
        const Tap ty = tys[r];
        const long long r0 = (long long)ty.i0 * J.spitch, r1 = (long long)ty.i1 * J.spitch;
        const long long o = (long long)(ybase + r) * J.dpitch + x;
        float a[NP], b[NP], c[NP], d[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float* s = J.src + p * J.spstride;
            a[p] = __ldg(s + r0 + tx.i0);
            b[p] = __ldg(s + r0 + tx.i1);
            c[p] = __ldg(s + r1 + tx.i0);
            d[p] = __ldg(s + r1 + tx.i1);
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) J.dst[p * J.dpstride + o] = bilerp(a[p], b[p], c[p], d[p], tx.t, ty.t);
    }
}

template <>
__device__ __forceinline__ void resample_tile<0>(const ResampleJob& J, int x, int ybase, const Tap* tys) {
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
        switch (J.nplanes) {
            case 1: resample_tile<1>(J, x, ybase, tys); break;
            case 3: resample_tile<3>(J, x, ybase, tys); break;
            case 6: resample_tile<6>(J, x, ybase, tys); break;
            default: resample_tile<0>(J, x, ybase, tys); break;
        }
    }
}

int resample_tiles(int dw, int dh) { return ((dw + kResCols - 1) / kResCols) * ((dh + kResRows - 1) / kResRows); }

cudaError_t launch_resample(const ResampleJob* jobs_dev, int njobs, long long total_tiles, cudaStream_t s) {
    if (njobs <= 0 || total_tiles <= 0) return cudaSuccess;
    const int gx = int(std::min<long long>(total_tiles, 148 * 16));
    resample_kernel<<<gx, kResCols, 0, s>>>(jobs_dev, njobs, int(total_tiles));
    return cudaGetLastError();
}

// ============================================================================
// K4: coarse levels.  One CTA per image.  Per level: resample I/alpha from
// full-res (global) and F/B from the previous level (shared), then
// `iterations` sweeps in place in shared memory along the wavefront
// t = x + y + 2k (pixel (x,y) of sweep k depends only on step t-1 values;
// pixels updated in one step are never read in that step -- DESIGN.md).
// ============================================================================
constexpr int kCoarseThreads = 256;

size_t coarse_smem_bytes() { return size_t(16) * kCoarseCap * sizeof(float); }

__device__ __forceinline__ void coarse_update(float* __restrict__ sI, float* __restrict__ sA, float* __restrict__ fb,
                                              int x, int y, int w, int h, float eps, float omega) {
    const int n = w * h;
    const int i = y * w + x;
    const int jL = x > 0 ? i - 1 : i, jR = x < w - 1 ? i + 1 : i;
    const int jU = y > 0 ? i - w : i, jD = y < h - 1 ? i + w : i;
    float I[3];
    float L[6], R[6], U[6], D[6], out[6];
#pragma unroll
    for (int c = 0; c < 3; ++c) I[c] = sI[c * n + i];
    const Coef co = pixel_coef(sA[i], sA[jL], sA[jR], sA[jU], sA[jD], I, eps, omega);
#pragma unroll
    for (int p = 0; p < 6; ++p) {
        L[p] = fb[p * n + jL];
        R[p] = fb[p * n + jR];
        U[p] = fb[p * n + jU];
        D[p] = fb[p * n + jD];
    }
    pixel_apply(co, L, R, U, D, out);
#pragma unroll
    for (int p = 0; p < 6; ++p) fb[p * n + i] = out[p];
}

__global__ void __launch_bounds__(kCoarseThreads) coarse_kernel(const CoarseJob* __restrict__ jobs, float eps,
                                                                 float omega) {
    extern __shared__ float sm[];
    const CoarseJob& J = jobs[blockIdx.x];
    const int cap = kCoarseCap;
    float* sI = sm;
    float* sA = sm + 3 * cap;
    float* sFB[2] = {sm + 4 * cap, sm + 10 * cap};
    const int W = J.W, H = J.H;
    const long long fps = (long long)W * H;
    int pw = 1, ph = 1;
    const int nlev = J.nlev;
    for (int l = 0; l < nlev; ++l) {
        const int w = J.lw[l], h = J.lh[l], K = J.lit[l];
        const int n = w * h, pn = pw * ph;
        float* cur = sFB[l & 1];
        const float* prv = sFB[(l & 1) ^ 1];
        const bool ident = (w == W && h == H);
        const bool same = (w == pw && h == ph);
        const double sxf = __ddiv_rn(double(W), double(w)), syf = __ddiv_rn(double(H), double(h));
        const double sxp = __ddiv_rn(double(pw), double(w)), syp = __ddiv_rn(double(ph), double(h));
        for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
            const int y = idx / w, x = idx - y * w;
            if (ident) {  // the last level resamples the original: identity copy
#pragma unroll
                for (int c = 0; c < 3; ++c) sI[c * n + idx] = J.img[c * fps + idx];
                sA[idx] = J.alpha[idx];
            } else {
                const Tap tx = make_tap_s(x, W, sxf), ty = make_tap_s(y, H, syf);
                const long long r0 = (long long)ty.i0 * W, r1 = (long long)ty.i1 * W;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float* s = c < 3 ? J.img + c * fps : J.alpha;
                    const float v = bilerp(__ldg(s + r0 + tx.i0), __ldg(s + r0 + tx.i1), __ldg(s + r1 + tx.i0),
                                           __ldg(s + r1 + tx.i1), tx.t, ty.t);
                    if (c < 3)
                        sI[c * n + idx] = v;
                    else
                        sA[idx] = v;
                }
            }
            if (l == 0) {  // F, B start as 1x1 zeros (multilevel.cpp:155-156)
#pragma unroll
                for (int p = 0; p < 6; ++p) cur[p * n + idx] = 0.0f;
            } else if (same) {
#pragma unroll
                for (int p = 0; p < 6; ++p) cur[p * n + idx] = prv[p * pn + idx];
            } else {
                const Tap tx = make_tap_s(x, pw, sxp), ty = make_tap_s(y, ph, syp);
                const int r0 = ty.i0 * pw, r1 = ty.i1 * pw;
#pragma unroll
                for (int p = 0; p < 6; ++p) {
                    const float* s = prv + p * pn;
                    cur[p * n + idx] = bilerp(s[r0 + tx.i0], s[r0 + tx.i1], s[r1 + tx.i0], s[r1 + tx.i1], tx.t, ty.t);
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
                J.lvl_fg[l][idx] = cur[idx];
                J.lvl_bg[l][idx] = cur[3 * n + idx];
            }
        }
        pw = w;
        ph = h;
    }
    const float* fin = sFB[(nlev - 1) & 1];
    const int n = pw * ph;
    for (int idx = threadIdx.x; idx < 3 * n; idx += blockDim.x) {
        const int c = idx / n, i = idx - c * n, y = i / pw, x = i - y * pw;
        const long long o = c * J.out_pstride + (long long)y * J.out_pitch + x;
        J.fg_out[o] = fin[idx];
        J.bg_out[o] = fin[3 * n + idx];
    }
}

cudaError_t launch_coarse(const CoarseJob* jobs_dev, int njobs, float eps, float omega, cudaStream_t s) {
    if (njobs <= 0) return cudaSuccess;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(coarse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(coarse_smem_bytes()));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
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
