// Host/device shared job descriptors and launch entry points of the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace fgm {

// ---- K1/K2: bilinear resample (image.cpp:71-133) --------------------------
struct ResampleJob {
    const float* src;
    float* dst;
    int sw, sh, dw, dh, nplanes;
    long long spstride, dpstride;  // plane strides in floats
};

// ---- K4: coarse levels, one CTA per image, shared-memory resident ---------
constexpr int kMaxCoarseLevels = 24;
constexpr int kCoarseCap = 2048;  // max pixels of a level handled by K4

struct CoarseJob {
    const float* img;  // full-res, 3 planes
    const float* alpha;
    int W, H;
    int nlev;
    int lw[kMaxCoarseLevels], lh[kMaxCoarseLevels], lit[kMaxCoarseLevels];
    float* fg_out;  // last coarse level F (3 planes, stride lw*lh)
    float* bg_out;
    float* lvl_fg[kMaxCoarseLevels];  // optional per-level dumps (debug API)
    float* lvl_bg[kMaxCoarseLevels];
};

// ---- K3: big-level sweep, skewed-band wavefront ---------------------------
constexpr int kBandRows = 32;   // one warp = 32 skewed rows
constexpr int kChunk = 32;      // boundary-stream publication granularity (columns)
constexpr int kWarpsPerCta = 4;

struct SweepJob {
    const float* img;    // 3 planes
    const float* alpha;  // 1 plane
    const float* fg_in;  // 3 planes (initial F of this pass)
    const float* bg_in;
    float* fg_out;
    float* bg_out;
    float* stream;       // nb * (w + K - 1) * K * 6 floats
    unsigned* progress;  // nb counters (zeroed before launch)
    long long pstride;   // w*h
    int w, h, nb, band_base;
};

inline int sweep_bands(int h, int K) { return (h + K - 1 + kBandRows - 1) / kBandRows; }
inline size_t sweep_stream_floats(int w, int h, int K) {
    return size_t(sweep_bands(h, K)) * size_t(w + K - 1) * size_t(K) * 6;
}

// Launch helpers (kernels.cu).  `jobs_dev` are device copies of the arrays.
cudaError_t launch_resample(const ResampleJob* jobs_dev, int njobs, long long max_px, cudaStream_t s);
cudaError_t launch_coarse(const CoarseJob* jobs_dev, int njobs, float eps, float omega, cudaStream_t s);
cudaError_t launch_sweep(int K, const SweepJob* jobs_dev, int njobs, int total_bands, unsigned* ticket, float eps,
                         float omega, cudaStream_t s);
cudaError_t launch_f64_to_f32(const double* src, float* dst, size_t n, cudaStream_t s);
cudaError_t launch_f32_to_f64(const float* src, double* dst, size_t n, cudaStream_t s);
size_t coarse_smem_bytes();
int sweep_supported_k(int K);  // 1 if a K-template exists

}  // namespace fgm
