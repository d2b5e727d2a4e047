// sm_100a kernels of the multi-level F/B estimator.
//
//   K1/K2 resample_kernel  -- bilinear level resampling (image.cpp:71-133)
//   K4    coarse_kernel    -- all coarse levels of an image in one CTA, in
//                             shared memory, exact Gauss-Seidel order
//   K3    sweep_kernel<K>  -- K fused in-place scanline sweeps of one big level
//                             (multilevel.cpp:81-121 x iterations), as a
//                             skewed-band wavefront across warps / CTAs
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
__global__ void __launch_bounds__(256) resample_kernel(const ResampleJob* __restrict__ jobs) {
    const ResampleJob J = jobs[blockIdx.y];
    const bool ident = (J.sw == J.dw && J.sh == J.dh);
    for (int y = blockIdx.x; y < J.dh; y += gridDim.x) {
        if (ident) {
            for (int x = threadIdx.x; x < J.dw; x += blockDim.x) {
                const long long i = (long long)y * J.dw + x;
                for (int p = 0; p < J.nplanes; ++p) J.dst[p * J.dpstride + i] = J.src[p * J.spstride + i];
            }
            continue;
        }
        const Tap ty = make_tap(y, J.sh, J.dh);
        for (int x = threadIdx.x; x < J.dw; x += blockDim.x) {
            const Tap tx = make_tap(x, J.sw, J.dw);
            const long long r0 = (long long)ty.i0 * J.sw, r1 = (long long)ty.i1 * J.sw;
            const long long o = (long long)y * J.dw + x;
            for (int p = 0; p < J.nplanes; ++p) {
                const float* s = J.src + p * J.spstride;
                J.dst[p * J.dpstride + o] =
                    bilerp(__ldg(s + r0 + tx.i0), __ldg(s + r0 + tx.i1), __ldg(s + r1 + tx.i0), __ldg(s + r1 + tx.i1),
                           tx.t, ty.t);
            }
        }
    }
}

cudaError_t launch_resample(const ResampleJob* jobs_dev, int njobs, long long max_rows, cudaStream_t s) {
    if (njobs <= 0) return cudaSuccess;
    const int gx = int(std::min<long long>(std::max<long long>(max_rows, 1), 2048));
    resample_kernel<<<dim3(gx, njobs), 256, 0, s>>>(jobs_dev);
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
    PixelIn P;
    P.a = sA[i];
    P.aL = sA[jL];
    P.aR = sA[jR];
    P.aU = sA[jU];
    P.aD = sA[jD];
    float L[6], R[6], U[6], D[6], out[6];
#pragma unroll
    for (int c = 0; c < 3; ++c) P.I[c] = sI[c * n + i];
#pragma unroll
    for (int p = 0; p < 6; ++p) {
        L[p] = fb[p * n + jL];
        R[p] = fb[p * n + jR];
        U[p] = fb[p * n + jU];
        D[p] = fb[p * n + jD];
    }
    solve_pixel(P, L, R, U, D, eps, omega, out);
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
        for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
            const int y = idx / w, x = idx - y * w;
            if (ident) {  // the last level resamples the original: identity copy
#pragma unroll
                for (int c = 0; c < 3; ++c) sI[c * n + idx] = J.img[c * fps + idx];
                sA[idx] = J.alpha[idx];
            } else {
                const Tap tx = make_tap(x, W, w), ty = make_tap(y, H, h);
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
                const Tap tx = make_tap(x, pw, w), ty = make_tap(y, ph, h);
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
        J.fg_out[idx] = fin[idx];
        J.bg_out[idx] = fin[3 * n + idx];
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
// K3: big-level sweeps.
//
// Skewed coordinates u = x + k, v = y + k turn every dependency of the
// in-place scanline Gauss-Seidel (L, U new; R, D, self old) into a
// non-negative (du, dv) step, so bands of 32 skewed rows depend only on the
// band above.  Lane j of a warp owns skewed row v = 32q + j; at step t it
// updates, for every sweep k < K, pixel (x, y) = (t - v - k, v - k).  All
// neighbour values come from the lane itself or from lane j-1 one step
// earlier (registers + shfl).  Lane 0 gets lane "-1" (the band above) from
// that band's boundary stream in global memory, published every kChunk
// columns with release/acquire counters.  Bands are handed out by an atomic
// ticket in dependency order, so every awaited band is already running.
// ============================================================================
template <int K>
__device__ __forceinline__ void run_band(const SweepJob& J, int q, int lane, float* __restrict__ chunk, float eps,
                                         float omega) {
    const int w = J.w, h = J.h;
    const int Umax = w + K - 1;
    const int v = q * kBandRows + lane;
    const long long ps = J.pstride;
    const float* __restrict__ A = J.alpha;
    const float* __restrict__ IM = J.img;
    const float* __restrict__ FI = J.fg_in;
    const float* __restrict__ BI = J.bg_in;
    float* __restrict__ FO = J.fg_out;
    float* __restrict__ BO = J.bg_out;
    const size_t slen = size_t(Umax) * K * 6;
    const float* up_stream = q > 0 ? J.stream + size_t(q - 1) * slen : nullptr;
    float* my_stream = J.stream + size_t(q) * slen;
    const bool has_down = q < J.nb - 1;
    const bool vrow = v < h;

    float outp[K][6], rprev[K][6];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < 6; ++c) outp[k][c] = rprev[k][c] = 0.0f;
    float fbR[6], fbS[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) fbR[c] = fbS[c] = 0.0f;
    float aR = 0.0f, aS = 0.0f, aL = 0.0f;

    const int tbeg = q * kBandRows - 1;
    const int tend = q * kBandRows + (kBandRows - 1) + Umax;
    for (int t = tbeg; t < tend; ++t) {
        const int u = t - v;
        const int u0 = t - q * kBandRows;  // lane 0's column
        if (q > 0 && u0 >= 0 && u0 < Umax && (u0 % kChunk) == 0) {
            const int need = min(u0 + kChunk, Umax);
            while (ld_acquire(J.progress + (q - 1)) < unsigned(need)) __nanosleep(32);
            __syncwarp();
            const int nfl = (need - u0) * K * 6;
            const float* src = up_stream + size_t(u0) * K * 6;
            for (int e = lane; e < nfl; e += 32) chunk[e] = __ldcg(src + e);
            __syncwarp();
        }
        // values of lane j-1 from step t-1: U of sweep k, R of sweep k+1
        float recv[K][6];
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int c = 0; c < 6; ++c) recv[k][c] = __shfl_up_sync(kFull, outp[k][c], 1);
        if (lane == 0) {
            const bool ok = q > 0 && u0 >= 0 && u0 < Umax;
            const float* src = chunk + (ok ? (u0 % kChunk) * K * 6 : 0);
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int c = 0; c < 6; ++c) recv[k][c] = ok ? src[k * 6 + c] : 0.0f;
        }
        // sweep 0 reads the pass input: slide (u, v) <- (u+1, v)
#pragma unroll
        for (int c = 0; c < 6; ++c) fbS[c] = fbR[c];
        aL = aS;
        aS = aR;
        {
            const int x1 = u + 1;
            if (vrow && x1 >= 0 && x1 < w) {
                const long long idx = (long long)v * w + x1;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    fbR[c] = __ldg(FI + c * ps + idx);
                    fbR[3 + c] = __ldg(BI + c * ps + idx);
                }
                aR = __ldg(A + idx);
            } else {
#pragma unroll
                for (int c = 0; c < 6; ++c) fbR[c] = 0.0f;
                aR = 0.0f;
            }
        }
        float fbD0[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) fbD0[c] = __shfl_down_sync(kFull, fbR[c], 1);
        float aD0 = __shfl_down_sync(kFull, aR, 1);
        float aU0 = __shfl_up_sync(kFull, aL, 1);
        if (lane == kBandRows - 1 && v + 1 < h && u >= 0 && u < w) {
            const long long idx = (long long)(v + 1) * w + u;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                fbD0[c] = __ldg(FI + c * ps + idx);
                fbD0[3 + c] = __ldg(BI + c * ps + idx);
            }
            aD0 = __ldg(A + idx);
        }
        if (lane == 0 && v >= 1 && v - 1 < h && u >= 0 && u < w) aU0 = __ldg(A + (long long)(v - 1) * w + u);

        float nv[K][6];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int x = u - k, y = v - k;
            const bool act = x >= 0 && x < w && y >= 0 && y < h;
            if (act) {
                const long long idx = (long long)y * w + x;
                PixelIn P;
                float self[6], L[6], R[6], U[6], D[6];
#pragma unroll
                for (int c = 0; c < 6; ++c) self[c] = k == 0 ? fbS[c] : rprev[k > 0 ? k - 1 : 0][c];
                if (k == 0) {
                    P.a = aS;
                    P.aL = x > 0 ? aL : aS;
                    P.aR = x < w - 1 ? aR : aS;
                    P.aU = y > 0 ? aU0 : aS;
                    P.aD = y < h - 1 ? aD0 : aS;
                } else {
                    P.a = __ldg(A + idx);
                    P.aL = x > 0 ? __ldg(A + idx - 1) : P.a;
                    P.aR = x < w - 1 ? __ldg(A + idx + 1) : P.a;
                    P.aU = y > 0 ? __ldg(A + idx - w) : P.a;
                    P.aD = y < h - 1 ? __ldg(A + idx + w) : P.a;
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) P.I[c] = __ldg(IM + c * ps + idx);
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    L[c] = x > 0 ? outp[k][c] : self[c];
                    R[c] = x < w - 1 ? (k == 0 ? fbR[c] : recv[k > 0 ? k - 1 : 0][c]) : self[c];
                    U[c] = y > 0 ? recv[k][c] : self[c];
                    D[c] = y < h - 1 ? (k == 0 ? fbD0[c] : outp[k > 0 ? k - 1 : 0][c]) : self[c];
                }
                solve_pixel(P, L, R, U, D, eps, omega, nv[k]);
                if (k == K - 1) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        FO[c * ps + idx] = nv[k][c];
                        BO[c * ps + idx] = nv[k][3 + c];
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < 6; ++c) nv[k][c] = 0.0f;
            }
        }
        if (lane == kBandRows - 1 && has_down && u >= 0 && u < Umax) {
            float* dst = my_stream + size_t(u) * K * 6;
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int c = 0; c < 6; ++c) dst[k * 6 + c] = nv[k][c];
            if (((u + 1) % kChunk) == 0 || u + 1 == Umax) {
                __threadfence();
                st_release(J.progress + q, unsigned(u + 1));
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                rprev[k][c] = recv[k][c];
                outp[k][c] = nv[k][c];
            }
    }
}

template <int K>
__global__ void __launch_bounds__(kWarpsPerCta * 32) sweep_kernel(const SweepJob* __restrict__ jobs, int njobs,
                                                                   int total_bands, unsigned* ticket, float eps,
                                                                   float omega) {
    __shared__ float chunks[kWarpsPerCta][kChunk * K * 6];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        unsigned tk = 0;
        if (lane == 0) tk = atomicAdd(ticket, 1u);
        tk = __shfl_sync(kFull, tk, 0);
        if (tk >= unsigned(total_bands)) return;
        int lo = 0, hi = njobs - 1;  // last job with band_base <= tk
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (unsigned(jobs[mid].band_base) <= tk)
                lo = mid;
            else
                hi = mid - 1;
        }
        const SweepJob J = jobs[lo];
        run_band<K>(J, int(tk) - J.band_base, lane, chunks[warp], eps, omega);
    }
}

template <int K>
static cudaError_t launch_sweep_k(const SweepJob* jobs_dev, int njobs, int total_bands, unsigned* ticket, float eps,
                                  float omega, cudaStream_t s) {
    static int grid_cap = 0;
    if (grid_cap == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<K>, kWarpsPerCta * 32, 0);
        grid_cap = std::max(1, sms * std::max(1, per_sm));
    }
    const int want = (total_bands + kWarpsPerCta - 1) / kWarpsPerCta;
    const int grid = std::max(1, std::min(want, grid_cap));
    sweep_kernel<K><<<grid, kWarpsPerCta * 32, 0, s>>>(jobs_dev, njobs, total_bands, ticket, eps, omega);
    return cudaGetLastError();
}

int sweep_supported_k(int K) { return K == 1 || K == 2 || K == 3 || K == 4 || K == 8; }

cudaError_t launch_sweep(int K, const SweepJob* jobs_dev, int njobs, int total_bands, unsigned* ticket, float eps,
                         float omega, cudaStream_t s) {
    switch (K) {
        case 1: return launch_sweep_k<1>(jobs_dev, njobs, total_bands, ticket, eps, omega, s);
        case 2: return launch_sweep_k<2>(jobs_dev, njobs, total_bands, ticket, eps, omega, s);
        case 3: return launch_sweep_k<3>(jobs_dev, njobs, total_bands, ticket, eps, omega, s);
        case 4: return launch_sweep_k<4>(jobs_dev, njobs, total_bands, ticket, eps, omega, s);
        case 8: return launch_sweep_k<8>(jobs_dev, njobs, total_bands, ticket, eps, omega, s);
        default: return cudaErrorInvalidValue;
    }
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
