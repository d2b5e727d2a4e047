// Host/device shared job descriptors and launch entry points of the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

namespace fgm {

// A lazily initialised value per CUDA device (function attributes, occupancy,
// memory pools are per device; a process may drive several GPUs from several
// host threads).  init(dev, value&) runs once per device under a lock.
template <class T>
class PerDevice {
   public:
    template <class F>
    cudaError_t get(T& out, F&& init) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev < 0 || dev >= kMax) return cudaErrorInvalidDevice;
        std::lock_guard<std::mutex> g(mu_);
        if (!ok_[dev]) {
            if ((e = init(dev, v_[dev])) != cudaSuccess) return e;
            ok_[dev] = true;
        }
        out = v_[dev];
        return cudaSuccess;
    }

   private:
    static constexpr int kMax = 64;
    std::mutex mu_;
    T v_[kMax]{};
    bool ok_[kMax] = {};
};

// ---- K1/K2: bilinear resample (image.cpp:71-133) --------------------------
struct ResampleJob {
    const float* src;
    float* dst;
    int sw, sh, dw, dh, nplanes;
    int spitch, dpitch;            // row strides in floats
    long long spstride, dpstride;  // plane strides in floats
    double sx, sy;                 // double(sw)/double(dw), double(sh)/double(dh) (image.cpp:73)
    int tile_base;                 // first tile of this job in the launch's flat tile space
    int idx32;                     // every src/dst element index fits in int32 (set by the host)
};

// ---- K1': the I/alpha pyramid of every big sub-top level of an image in one
// pass over the full-resolution input (image.cpp:114-133 per level) ---------
constexpr int kMaxPyr = 12;
constexpr int kPyrTH = 16, kPyrTW = 128;  // full-res tile (plus one overlap row and column)

struct PyrJob {
    const float* img;    // full-res, 3 planes, dense
    const float* alpha;
    int W, H;
    int nlev;
    int tile_base;       // first tile of this job in the launch's flat tile space
    int tcols;           // tiles per full-res tile row
    int lw[kMaxPyr], lh[kMaxPyr], pitch[kMaxPyr];
    double sx[kMaxPyr], sy[kMaxPyr];    // double(W)/double(lw), double(H)/double(lh) (image.cpp:73)
    double rsx[kMaxPyr], rsy[kMaxPyr];  // their reciprocals (tile-range estimates only)
    float* out[kMaxPyr];  // 4 pitched planes I0, I1, I2, alpha (plane stride pitch * lh)
};
inline int pyramid_tiles(int W, int H) { return ((W + kPyrTW - 1) / kPyrTW) * ((H + kPyrTH - 1) / kPyrTH); }
cudaError_t launch_pyramid(const PyrJob* jobs_dev, int njobs, long long total_tiles, cudaStream_t s);

// ---- K4: coarse levels, one CTA per image, shared-memory resident, fp64 ----
constexpr int kMaxCoarseLevels = 24;
constexpr int kCoarseCap = 1024;  // max pixels of a level handled by K4 (every level with max(w, h) <= 32)

struct CoarseJob {
    const float* img;  // full-res, 3 planes
    const float* alpha;
    const double* img64;  // optional fp64 full-res input (the fp64 host path), used instead of img/alpha
    const double* alpha64;
    int W, H;
    int nlev;
    int lw[kMaxCoarseLevels], lh[kMaxCoarseLevels], lit[kMaxCoarseLevels];
    float* fg_out;  // last coarse level F (3 planes)
    float* bg_out;
    double* fg_out64;  // optional: the same in fp64 (fp64 host path, image entirely coarse)
    double* bg_out64;
    int out_pitch;         // row stride of fg_out / bg_out
    long long out_pstride; // plane stride of fg_out / bg_out
    float* lvl_fg[kMaxCoarseLevels];  // optional per-level dumps (debug API)
    float* lvl_bg[kMaxCoarseLevels];
};

// ---- K3: big-level sweep, skewed-band wavefront ---------------------------
constexpr int kBandRows = 64;     // throughput kernel (sweep.cu): one warp = 64 skewed rows, two per lane
constexpr int kLatBandRows = 32;  // latency kernel (sweep_ws.cu): one CTA = 32 skewed rows, one per lane of a chain warp
constexpr int kLatMaxJobs = 4;    // launches of at most this many images are chain-bound: latency kernel
#ifndef FGM_CHUNK
#define FGM_CHUNK 16
#endif
constexpr int kChunk = FGM_CHUNK;  // boundary-stream polling granularity (columns)
constexpr unsigned kStreamSentinel = 0xFFFFFFFFu;  // a NaN: never a clamped output

struct SweepJob {
    const float* img;    // 3 planes
    const float* alpha;  // 1 plane
    const float* fg_in;  // 3 planes (initial F of this pass)
    const float* bg_in;
    float* fg_out;
    float* bg_out;
    float* stream;       // 3 * nb streams of sweep_stream_len(w, K) floats, sentinel-filled before launch
    long long istride, fstride, ostride;  // plane strides: img/alpha, fg_in/bg_in, fg_out/bg_out
    int ipitch, fpitch, opitch;           // row strides of the same
    int w, h, nb, band_base;
    int vec4;            // all input rows 16-byte aligned (pitches % 4 == 0, aligned bases): 16-byte cp.async
};

// A job of one sweep launch is split into (band, channel) work items: band q,
// channel c has stream / counter index 3q + c.  A stream holds, per skewed
// column u, the K (F_c, B_c) pairs of the band's last row, padded to 16 bytes.
// Row pitch of the solver's own level buffers: whole 16-byte blocks, so the
// sweep streams them with 16-byte cp.async whatever the level width.
inline int level_pitch(int w) { return (w + 3) & ~3; }

inline int sweep_bands(int h, int K, int rows = kBandRows) { return (h + K - 1 + rows - 1) / rows; }
__host__ __device__ inline size_t sweep_stream_len(int w, int K) {
    return (size_t(w + K - 1) * size_t(K) * 2 + 3) / 4 * 4;
}
inline size_t sweep_stream_floats(int w, int h, int K, int rows = kBandRows) {
    return size_t(sweep_bands(h, K, rows)) * 3 * sweep_stream_len(w, K);
}
// Launch helpers (kernels.cu).  `jobs_dev` are device copies of the arrays.
// Tiles of 128 x 8 destination pixels; total_tiles = sum over jobs.
int resample_tiles(int dw, int dh);
// blocks_per_sm: persistent grid size (16 fills the GPU; the side-stream
// pyramid uses fewer so the main stream's kernels can co-reside)
cudaError_t launch_resample(const ResampleJob* jobs_dev, int njobs, long long total_tiles, cudaStream_t s,
                            int blocks_per_sm = 16);
// F/B upsample (sw <= dw, sh <= dh, six planes): shared-memory staged tiles
int upsample_tiles(int dw, int dh);
cudaError_t launch_upsample(const ResampleJob* jobs_dev, int njobs, long long total_tiles, cudaStream_t s);
bool upsample_ok(int sw, int sh, int dw, int dh);
cudaError_t launch_hwc_to_planar(const void* src, bool f64, long long n, int ch, float* dst, cudaStream_t s);
cudaError_t launch_planar_to_hwc(const float* src, long long n, int ch, void* dst, bool f64, cudaStream_t s);
int metrics_blocks(long long n);
cudaError_t launch_metrics(const float* est, const float* gt, const float* alpha, int w, int h, int nch,
                           const double* kern, int r, double* partial, int blocks, cudaStream_t s);
cudaError_t launch_compose(const float* fg, const float* bg, const float* alpha, long long n, int nch, float* out,
                           cudaStream_t s);  // scale within the staged window
cudaError_t launch_coarse(const CoarseJob* jobs_dev, int njobs, double eps, double omega, cudaStream_t s);
// order_dev[t] = (job, 3 * band + channel) of ticket t, band-major across jobs.
// ticket: the launch's zeroed ticket counter; abort_flag: a zeroed per-launch
// int (a timed-out boundary-stream wait sets it and every waiter gives up);
// fault_count: a persistent per-device counter of timed-out waits.
cudaError_t launch_sweep(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket,
                         float eps, float omega, int* abort_flag, int* fault_count, cudaStream_t s);
// The same for jobs cut into kLatBandRows-row bands: the warp-specialised
// latency kernel (sweep_ws.cu), one CTA per band -- two producer warps compute
// the alpha-only coefficients once per pixel, one chain warp per channel runs
// the recurrence, one helper warp per channel streams the rings and flushes
// the outputs.  Same jobs, order and streams (three items per band).
cudaError_t launch_sweep_ws(int K, const SweepJob* jobs_dev, const int2* order_dev, int total_items, unsigned* ticket,
                            float eps, float omega, int* abort_flag, int* fault_count, cudaStream_t s);
extern std::atomic<int> g_sweep_fault;            // debug fault injection (fgm_debug_fault)
extern std::atomic<long long> g_spin_timeout_ns;  // bound on one boundary-stream wait
// Fill every job's boundary streams with kStreamSentinel (before its sweep).
cudaError_t launch_stream_fill(const SweepJob* jobs_dev, int njobs, int K, size_t max_floats, cudaStream_t s);
cudaError_t launch_f64_to_f32(const double* src, float* dst, size_t n, cudaStream_t s);
cudaError_t launch_f32_to_f64(const float* src, double* dst, size_t n, cudaStream_t s);
size_t coarse_smem_bytes();
int sweep_supported_k(int K);  // 1 if a K-template exists
size_t sweep_smem_bytes(int K);

}  // namespace fgm
