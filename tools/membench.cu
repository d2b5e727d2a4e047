// Memory-staging microbenchmark for the K3 redesign (development tool, not
// part of the library): sustained HBM->SM bandwidth of the access patterns a
// row-band sweep can use to stage its rows, and of its output patterns.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu
//   tools/membench
//
// Every warp owns a band of 32 rows of a 2 GiB plane and streams all of its
// columns.  Load modes keep about the same bytes in flight per warp:
//   cpasync<LPR>: cp.async 16 B per lane, LPR consecutive lanes per row
//                 (one instruction covers 32/LPR rows x 16*LPR bytes)
//   bulk<S>:      one cp.async.bulk of S bytes per row (lane = row), mbarrier
//   ldg<LPR>:     LDG.128 into registers, LPR lanes per row
// Store modes:
//   stg128_rows:  STG.128, lane = row (32 rows x 16 B per instruction)
//   stg32_2rows:  STG.32, lanes 0-15 row a, 16-31 row b (2 x 64 B)
//   stg128<LPR>:  STG.128, LPR lanes per row
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess) {                                                        \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

constexpr int W = 8192;        // floats per row
constexpr int H = 65536;       // rows (2 GiB)
constexpr int INFLIGHT = 8192;  // bytes in flight per warp

extern __shared__ float4 sm4[];

__device__ __forceinline__ void cp16(unsigned s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}

template <int LPR>
__global__ void __launch_bounds__(32) k_cpasync(const float* __restrict__ src, float* out) {
    constexpr int SEG = 4 * LPR;                  // floats per row per stage
    constexpr int NST = INFLIGHT / (32 * SEG * 4);  // stages in flight
    constexpr int RPI = 32 / LPR;                 // rows per instruction
    const int lane = threadIdx.x;
    const int band = blockIdx.x;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(sm4);
    // smem: [2*NST stages][32 rows][SEG]
    float acc = 0.f;
    const int nsteps = W / SEG;
    auto issue = [&](int st) {
        const int slot = st % (2 * NST);
#pragma unroll
        for (int q = 0; q < LPR; ++q) {
            const int r = q * RPI + lane / LPR;
            const int c = (lane % LPR) * 4;
            const float* g = src + (size_t)(band * 32 + r) * W + st * SEG + c;
            cp16(sb + 4u * (unsigned)((slot * 32 + r) * SEG + c), g);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int st = 0; st < NST; ++st) issue(st);
    const float* smf = reinterpret_cast<const float*>(sm4);
    for (int st = 0; st < nsteps; ++st) {
        if (st + NST < nsteps)
            issue(st + NST);
        else
            asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(NST) : "memory");
        __syncwarp();
        const int slot = st % (2 * NST);
        acc += smf[(slot * 32 + lane) * SEG + (st & (SEG - 1))];
    }
    if (acc == 12345.f) out[band] = acc;
}

template <int S>  // bytes per row per stage
__global__ void __launch_bounds__(32) k_bulk(const float* __restrict__ src, float* out) {
    constexpr int SEG = S / 4;
    constexpr int NST = INFLIGHT / (32 * S) > 0 ? INFLIGHT / (32 * S) : 1;
    constexpr int NS2 = 2 * NST;
    const int lane = threadIdx.x;
    const int band = blockIdx.x;
    __shared__ __align__(8) unsigned long long bar[2 * 16];
    const unsigned sb = (unsigned)__cvta_generic_to_shared(sm4);
    if (lane < NS2) {
        unsigned b = (unsigned)__cvta_generic_to_shared(&bar[lane]);
        asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(b), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int nsteps = W / SEG;
    auto issue = [&](int st) {
        const int slot = st % NS2;
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[slot]);
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(32 * S) : "memory");
        __syncwarp();
        const float* g = src + (size_t)(band * 32 + lane) * W + st * SEG;
        const unsigned d = sb + 4u * (unsigned)((slot * 32 + lane) * SEG);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                     "l"(g), "r"(S), "r"(b)
                     : "memory");
    };
    for (int st = 0; st < NST && st < nsteps; ++st) issue(st);
    const float* smf = reinterpret_cast<const float*>(sm4);
    float acc = 0.f;
    for (int st = 0; st < nsteps; ++st) {
        const int slot = st % NS2;
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[slot]);
        const unsigned parity = (st / NS2) & 1;
        asm volatile(
            "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(b),
            "r"(parity)
            : "memory");
        acc += smf[(slot * 32 + lane) * SEG + (st & (SEG - 1))];
        __syncwarp();
        if (st + NST < nsteps) issue(st + NST);
    }
    if (acc == 12345.f) out[band] = acc;
}

template <int LPR>
__global__ void __launch_bounds__(32) k_ldg(const float* __restrict__ src, float* out) {
    constexpr int SEG = 4 * LPR;
    constexpr int RPI = 32 / LPR;
    constexpr int U = INFLIGHT / (32 * 16);  // LDG.128 in flight per lane
    const int lane = threadIdx.x;
    const int band = blockIdx.x;
    float acc = 0.f;
    const int nsteps = W / SEG;  // per row group
    for (int q = 0; q < LPR; ++q) {
        const int r = q * RPI + lane / LPR;
        const float4* g = reinterpret_cast<const float4*>(src + (size_t)(band * 32 + r) * W + (lane % LPR) * 4);
        for (int st = 0; st < nsteps; st += U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcg(g + (size_t)(st + u) * LPR);
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
        }
    }
    if (acc == 12345.f) out[band] = acc;
}

template <int LPR>
__global__ void __launch_bounds__(32) k_stg128(float* dst) {
    constexpr int SEG = 4 * LPR;
    constexpr int RPI = 32 / LPR;
    const int lane = threadIdx.x;
    const int band = blockIdx.x;
    const int nsteps = W / SEG;
    const float4 v = make_float4(lane, 1.f, 2.f, 3.f);
    for (int st = 0; st < nsteps; ++st) {
#pragma unroll
        for (int q = 0; q < LPR; ++q) {
            const int r = q * RPI + lane / LPR;
            float4* g = reinterpret_cast<float4*>(dst + (size_t)(band * 32 + r) * W + st * SEG + (lane % LPR) * 4);
            __stcg(g, v);
        }
    }
}

__global__ void __launch_bounds__(32) k_stg32_2rows(float* dst) {
    const int lane = threadIdx.x;
    const int band = blockIdx.x;
    // per step: rows (2s, 2s+1) mod 32 get a 16-column segment at column 16*seg
    const int nseg = W / 16;
    for (int sgi = 0; sgi < nseg; ++sgi)
        for (int rp = 0; rp < 16; ++rp) {
            const int r = 2 * rp + (lane >> 4);
            dst[(size_t)(band * 32 + r) * W + sgi * 16 + (lane & 15)] = float(lane);
        }
}

template <typename F>
double run(const char* name, F launch, double bytes) {
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
    const double gbs = bytes * reps / (ms * 1e-3) / 1e9;
    printf("%-22s %8.3f ms  %8.1f GB/s\n", name, ms / reps, gbs);
    return gbs;
}

int main() {
    float *src, *dst, *out;
    const size_t n = (size_t)W * H;
    CK(cudaMalloc(&src, n * 4));
    CK(cudaMalloc(&dst, n * 4));
    CK(cudaMalloc(&out, 65536 * 4));
    CK(cudaMemset(src, 0, n * 4));
    const int grid = H / 32;
    const double bytes = double(n) * 4;
    int dev = 0, sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    printf("membench: %d SMs, plane %zu MB, %d warps (one 32-row band each), %d B in flight per warp\n", sms,
           n * 4 >> 20, grid, INFLIGHT);
    const size_t smc = 2 * INFLIGHT;
#define CPA(L)                                                                                          \
    CK(cudaFuncSetAttribute(k_cpasync<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc));     \
    run("cpasync lpr=" #L, [&] { k_cpasync<L><<<grid, 32, smc>>>(src, out); }, bytes);
    CPA(1) CPA(2) CPA(4) CPA(8)
#define BLK(S)                                                                                          \
    {                                                                                                   \
        const size_t sm = (size_t)2 * (INFLIGHT / (32 * S) > 0 ? INFLIGHT / (32 * S) : 1) * 32 * S;     \
        CK(cudaFuncSetAttribute(k_bulk<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));      \
        run("bulk S=" #S, [&] { k_bulk<S><<<grid, 32, sm>>>(src, out); }, bytes);                        \
    }
    BLK(16) BLK(32) BLK(64) BLK(128) BLK(256)
#define LDG(L) run("ldg128 lpr=" #L, [&] { k_ldg<L><<<grid, 32>>>(src, out); }, bytes);
    LDG(1) LDG(2) LDG(4) LDG(8)
#define STG(L) run("stg128 lpr=" #L, [&] { k_stg128<L><<<grid, 32>>>(dst); }, bytes);
    STG(1) STG(2) STG(4) STG(8)
    run("stg32 2rows x 64B", [&] { k_stg32_2rows<<<grid, 32>>>(dst); }, bytes);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return 0;
}
