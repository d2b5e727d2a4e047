// Device-side building blocks shared by the kernels: the per-pixel 2x2 solve
// and the exact bilinear taps.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fgm {

constexpr unsigned kFull = 0xffffffffu;

// Exact reference taps (image.cpp:71-83) computed in fp64 with explicit
// round-to-nearest intrinsics, so that no FMA contraction changes the result:
// bitwise the same (i0, i1, t) as the host code.  t is then rounded to fp32.
struct Tap {
    int i0, i1;
    float t;
};

__device__ __forceinline__ Tap make_tap(int d, int src, int dst) {
    const double scale = __ddiv_rn(double(src), double(dst));
    double f = __dadd_rn(__dmul_rn(__dadd_rn(double(d), 0.5), scale), -0.5);
    if (f < 0.0) f = 0.0;
    const double max_f = double(src - 1);
    if (f > max_f) f = max_f;
    const int i0 = int(f);
    Tap tp;
    tp.i0 = i0;
    tp.i1 = min(i0 + 1, src - 1);
    tp.t = float(__dadd_rn(f, -double(i0)));
    return tp;
}

// Two-stage lerp as resize_plane (image.cpp:98-102): horizontal on both rows,
// then vertical, then clamp01.
__device__ __forceinline__ float bilerp(float a, float b, float c, float d, float tx, float ty) {
    const float top = fmaf(tx, b - a, a);
    const float bot = fmaf(tx, d - c, c);
    return __saturatef(fmaf(ty, bot - top, top));
}

// dalpha = eps_r + omega * |alpha_i - alpha_j| (multilevel.cpp:106).
__device__ __forceinline__ float edge_weight(float ai, float aj, float eps, float omega) {
    return fmaf(omega, fabsf(ai - aj), eps);
}

// The per-pixel system of multilevel.cpp:94-118 (PixelSystem,
// multilevel.hpp:45-75), solved in a cancellation-free form.  With
// u = (a, 1-a), S = sum_j d_j, SF_c = sum_j d_j F_j,c, SB_c likewise,
// m = S^-1 * (SF, SB), the reference's adj(A) b / det(A) equals
//   F_c = (u1 (u1 mF - u0 mB) + u0 I_c + SF_c) / (u0^2 + u1^2 + S)
//   B_c = (u0 (u0 mB - u1 mF) + u1 I_c + SB_c) / (u0^2 + u1^2 + S)
// exactly in real arithmetic (det = S (u0^2 + u1^2 + S)).  In fp32 the
// reference's form loses ~log10(1/S) digits to cancellation (2e-3 max error at
// eps_r = 1e-5 on a 1x1 image); this form stays within a few ulps.  Every
// operation is written index-symmetrically in (F, B) / (u0, u1), so
// complementing alpha swaps the outputs bitwise (test_multilevel.cpp:167-180).
// Neighbour order L, R, U, D as multilevel.cpp:104-105.
struct PixelIn {
    float a, aL, aR, aU, aD;
    float I[3];
};

__device__ __forceinline__ void solve_pixel(const PixelIn& p, const float* L, const float* R, const float* U,
                                            const float* D, float eps, float omega, float* out) {
    const float dL = edge_weight(p.a, p.aL, eps, omega);
    const float dR = edge_weight(p.a, p.aR, eps, omega);
    const float dU = edge_weight(p.a, p.aU, eps, omega);
    const float dD = edge_weight(p.a, p.aD, eps, omega);
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(dL, dR), dU), dD);
    const float u0 = p.a;
    const float u1 = __fsub_rn(1.0f, p.a);
    const float iS = __frcp_rn(S);
    const float iD = __frcp_rn(__fadd_rn(__fadd_rn(__fmul_rn(u0, u0), __fmul_rn(u1, u1)), S));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float SF = __fmul_rn(dL, L[c]);
        float SB = __fmul_rn(dL, L[3 + c]);
        SF = __fmaf_rn(dR, R[c], SF);
        SB = __fmaf_rn(dR, R[3 + c], SB);
        SF = __fmaf_rn(dU, U[c], SF);
        SB = __fmaf_rn(dU, U[3 + c], SB);
        SF = __fmaf_rn(dD, D[c], SF);
        SB = __fmaf_rn(dD, D[3 + c], SB);
        const float mF = __fmul_rn(SF, iS);
        const float mB = __fmul_rn(SB, iS);
        const float tF = __fmaf_rn(u1, mF, -__fmul_rn(u0, mB));
        const float tB = __fmaf_rn(u0, mB, -__fmul_rn(u1, mF));
        out[c] = __saturatef(__fmul_rn(__fmaf_rn(u1, tF, __fmaf_rn(u0, p.I[c], SF)), iD));
        out[3 + c] = __saturatef(__fmul_rn(__fmaf_rn(u0, tB, __fmaf_rn(u1, p.I[c], SB)), iD));
    }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace fgm
