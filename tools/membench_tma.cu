// TMA box-load microbenchmark for the K3 redesign (development tool): HBM->smem
// bandwidth of 2D tiled TMA loads of narrow boxes (BW columns x BH rows,
// fp32), each warp (a 1-warp CTA) streaming a band of 64 rows of a 2 GiB
// plane, INFL bytes in flight per warp, OCC warps per SM (shared-memory
// sized), one mbarrier per stage.  Compared with cp.async of 64-byte row
// segments (4 lanes x 16 B per row) at the same occupancy.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench_tma tools/membench_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

constexpr int W = 8192;
constexpr int H = 65536;
constexpr int BAND = 64;

extern __shared__ __align__(128) unsigned char smraw[];

__device__ __forceinline__ void mbar_init(unsigned b, int n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void mbar_expect(unsigned b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(b), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma2d(unsigned dst, const CUtensorMap* m, int c0, int c1, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(m), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// stage = BAND rows x BW columns (BAND/BH boxes); NST stages in flight, 2*NST slots
template <int BW, int BH, int NST>
__global__ void __launch_bounds__(32) k_tma(const __grid_constant__ CUtensorMap map, float* out) {
    constexpr int NB = BAND / BH;
    constexpr unsigned STAGE = BAND * BW * 4;
    constexpr int NS2 = 2 * NST;
    const int lane = threadIdx.x;
    const int band = blockIdx.x;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smraw);
    float* data = reinterpret_cast<float*>(smraw + 256);
    const unsigned sb = (unsigned)__cvta_generic_to_shared(data);
    const unsigned bb = (unsigned)__cvta_generic_to_shared(bars);
    if (lane < NS2) mbar_init(bb + 8 * lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int nsteps = W / BW;
    auto issue = [&](int st) {
        const int slot = st % NS2;
        if (lane == 0) mbar_expect(bb + 8 * slot, STAGE);
        __syncwarp();
        if (lane < NB) tma2d(sb + slot * STAGE + lane * BH * BW * 4, &map, st * BW, band * BAND + lane * BH, bb + 8 * slot);
    };
    for (int st = 0; st < NST; ++st) issue(st);
    float acc = 0.f;
    for (int st = 0; st < nsteps; ++st) {
        const int slot = st % NS2;
        mbar_wait(bb + 8 * slot, (st / NS2) & 1);
        acc += data[slot * (STAGE / 4) + lane * BW + (st & (BW - 1))];
        __syncwarp();
        if (st + NST < nsteps) issue(st + NST);
    }
    if (acc == 12345.f) out[band] = acc;
}

// cp.async, 4 lanes x 16 B per row (64-byte row segments), stage = BAND rows x 16 columns
template <int NST>
__global__ void __launch_bounds__(32) k_cp64(const float* __restrict__ src, float* out) {
    constexpr int BW = 16;
    constexpr int NS2 = 2 * NST;
    const int lane = threadIdx.x;
    const int band = blockIdx.x;
    float* data = reinterpret_cast<float*>(smraw);
    const unsigned sb = (unsigned)__cvta_generic_to_shared(data);
    const int nsteps = W / BW;
    auto issue = [&](int st) {
        const int slot = st % NS2;
#pragma unroll
        for (int q = 0; q < BAND / 8; ++q) {
            const int r = q * 8 + lane / 4;
            const int c = (lane & 3) * 4;
            const float* g = src + (size_t)(band * BAND + r) * W + st * BW + c;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + 4u * (unsigned)(slot * BAND * BW + r * BW + c)),
                         "l"(g)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int st = 0; st < NST; ++st) issue(st);
    float acc = 0.f;
    for (int st = 0; st < nsteps; ++st) {
        if (st + NST < nsteps)
            issue(st + NST);
        else
            asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(NST) : "memory");
        __syncwarp();
        const int slot = st % NS2;
        acc += data[slot * BAND * BW + lane * BW + (st & (BW - 1))];
        __syncwarp();
    }
    if (acc == 12345.f) out[band] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename F>
void run(const char* name, F launch, double bytes) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch();
    CK(cudaDeviceSynchronize());
    const int reps = 3;
    CK(cudaEventRecord(a));
    for (int i = 0; i < reps; ++i) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-34s %8.3f ms  %8.1f GB/s\n", name, ms / reps, bytes * reps / (ms * 1e-3) / 1e9);
}

int main() {
    float *src, *out;
    const size_t n = (size_t)W * H;
    CK(cudaMalloc(&src, n * 4));
    CK(cudaMalloc(&out, 65536 * 4));
    CK(cudaMemset(src, 0, n * 4));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    const int grid = H / BAND;
    const double bytes = double(n) * 4;
    auto make = [&](int bw, int bh) {
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
        cuuint64_t strides[1] = {(cuuint64_t)W * 4};
        cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)r);
            exit(1);
        }
        return m;
    };
    printf("membench_tma: %d warps, band %d rows, plane %zu MB\n", grid, BAND, n * 4 >> 20);
    // smem sized to set the occupancy: occ warps/SM
    auto smem_for = [](int occ) { return (size_t)(220 * 1024 / occ) & ~(size_t)1023; };
#define TMA(BW, BH, NST, OCC)                                                                                  \
    {                                                                                                          \
        CUtensorMap m = make(BW, BH);                                                                          \
        size_t sm = smem_for(OCC);                                                                             \
        if (sm < 256 + 2 * NST * BAND * BW * 4) sm = 256 + 2 * NST * BAND * BW * 4;                            \
        CK(cudaFuncSetAttribute(k_tma<BW, BH, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));   \
        char nm[64];                                                                                           \
        snprintf(nm, 64, "tma box %dx%d nst=%d occ=%d", BW, BH, NST, OCC);                                     \
        run(nm, [&] { k_tma<BW, BH, NST><<<grid, 32, sm>>>(m, out); }, bytes);                                 \
    }
#define CP(NST, OCC)                                                                                           \
    {                                                                                                          \
        size_t sm = smem_for(OCC);                                                                             \
        if (sm < (size_t)2 * NST * BAND * 16 * 4) sm = 2 * NST * BAND * 16 * 4;                                \
        CK(cudaFuncSetAttribute(k_cp64<NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));          \
        char nm[64];                                                                                           \
        snprintf(nm, 64, "cp.async 64B rows nst=%d occ=%d", NST, OCC);                                         \
        run(nm, [&] { k_cp64<NST><<<grid, 32, sm>>>(src, out); }, bytes);                                      \
    }
    // 4 KB stages (64 rows x 16 cols)
    TMA(16, 4, 2, 14) TMA(16, 8, 2, 14) TMA(16, 16, 2, 14) TMA(16, 64, 2, 14)
    TMA(16, 4, 3, 5) TMA(16, 8, 3, 5) TMA(16, 16, 3, 5) TMA(16, 64, 3, 5)
    TMA(16, 4, 4, 5) TMA(16, 4, 6, 5)
    TMA(32, 4, 2, 5) TMA(32, 16, 2, 5)
    CP(2, 14) CP(3, 5) CP(4, 5) CP(6, 5)
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return 0;
}
