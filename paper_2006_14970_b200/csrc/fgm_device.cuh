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

// `scale` must be double(src) / double(dst), rounded (computed once per
// axis on the host, or by make_tap below).
__device__ __forceinline__ Tap make_tap_s(int d, int src, double scale) {
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

__device__ __forceinline__ Tap make_tap(int d, int src, int dst) {
    return make_tap_s(d, src, __ddiv_rn(double(src), double(dst)));
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
// multilevel.hpp:45-75).  With u = (a, 1-a), d_j = eps + omega |a - a_j| over
// the clamped neighbours L, R, U, D (multilevel.cpp:104-106), S = sum d_j and
// D = u0^2 + u1^2 + S, the reference's adj(A) b / det(A) (det = S D) equals
//   F_c = A  SF_c + Bc SB_c + (u0/D) I_c,   A  = (1 + u1^2/S) / D
//   B_c = A' SB_c + Bc SF_c + (u1/D) I_c,   A' = (1 + u0^2/S) / D,  Bc = -u0 u1 / (S D)
// with SF_c = sum_j d_j F_j,c (likewise SB_c).  The reference's form
// (diag1 rhs0 - off rhs1) / det cancels catastrophically in fp32 when S is
// small (2e-3 max error at eps_r = 1e-5 on a 1x1 image); this one has no
// cancellation beyond the data's own and stays within a few ulps of fp64.
// The alpha-only coefficients (Coef) are computed once per pixel; the
// neighbour part costs 4 FMAs per sum and 2 per output.  Every operation is
// mirrored in (F, B) / (u0, u1), so complementing alpha swaps the outputs
// bitwise (test_multilevel.cpp:167-180).  A clamped (missing) neighbour is
// passed as a_j = a, giving d_j = eps exactly as the reference's self term.
struct Coef {
    float dL, dR, dU, dD, A, A2, Bc, pI[3], qI[3];
};

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ Coef pixel_coef(float a, float aL, float aR, float aU, float aD, const float* I,
                                           float eps, float omega) {
    Coef co;
    co.dL = edge_weight(a, aL, eps, omega);
    co.dR = edge_weight(a, aR, eps, omega);
    co.dU = edge_weight(a, aU, eps, omega);
    co.dD = edge_weight(a, aD, eps, omega);
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(co.dL, co.dR), co.dU), co.dD);
    const float u0 = a, u1 = __fsub_rn(1.0f, a);
    const float u00 = __fmul_rn(u0, u0), u11 = __fmul_rn(u1, u1), u01 = __fmul_rn(u0, u1);
    const float iS = rcp_approx(S);
    const float iD = rcp_approx(__fadd_rn(__fadd_rn(u00, u11), S));
    co.A = __fmul_rn(iD, __fmaf_rn(u11, iS, 1.0f));
    co.A2 = __fmul_rn(iD, __fmaf_rn(u00, iS, 1.0f));
    co.Bc = -__fmul_rn(iD, __fmul_rn(u01, iS));
    const float p = __fmul_rn(iD, u0), qq = __fmul_rn(iD, u1);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        co.pI[c] = __fmul_rn(p, I[c]);
        co.qI[c] = __fmul_rn(qq, I[c]);
    }
    return co;
}

// Single-channel variants (one colour channel c; the sweep kernel runs the
// three channels in separate warps).
struct Coef1 {
    float dL, dR, dU, dD, A, A2, Bc, pI, qI;
};

__device__ __forceinline__ Coef1 pixel_coef1(float a, float aL, float aR, float aU, float aD, float I, float eps,
                                             float omega) {
    Coef1 co;
    co.dL = edge_weight(a, aL, eps, omega);
    co.dR = edge_weight(a, aR, eps, omega);
    co.dU = edge_weight(a, aU, eps, omega);
    co.dD = edge_weight(a, aD, eps, omega);
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(co.dL, co.dR), co.dU), co.dD);
    const float u0 = a, u1 = __fsub_rn(1.0f, a);
    const float u00 = __fmul_rn(u0, u0), u11 = __fmul_rn(u1, u1), u01 = __fmul_rn(u0, u1);
    const float iS = rcp_approx(S);
    const float iD = rcp_approx(__fadd_rn(__fadd_rn(u00, u11), S));
    co.A = __fmul_rn(iD, __fmaf_rn(u11, iS, 1.0f));
    co.A2 = __fmul_rn(iD, __fmaf_rn(u00, iS, 1.0f));
    co.Bc = -__fmul_rn(iD, __fmul_rn(u01, iS));
    co.pI = __fmul_rn(__fmul_rn(iD, u0), I);
    co.qI = __fmul_rn(__fmul_rn(iD, u1), I);
    return co;
}

// pixel_coef1 with the left edge weight given (the right edge weight of the
// left neighbour: |a - aL| is exactly symmetric, so it is the same value).
__device__ __forceinline__ Coef1 pixel_coef1_dl(float a, float dL, float aR, float aU, float aD, float I, float eps,
                                                float omega) {
    Coef1 co;
    co.dL = dL;
    co.dR = edge_weight(a, aR, eps, omega);
    co.dU = edge_weight(a, aU, eps, omega);
    co.dD = edge_weight(a, aD, eps, omega);
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(co.dL, co.dR), co.dU), co.dD);
    const float u0 = a, u1 = __fsub_rn(1.0f, a);
    const float u00 = __fmul_rn(u0, u0), u11 = __fmul_rn(u1, u1), u01 = __fmul_rn(u0, u1);
    const float iS = rcp_approx(S);
    const float iD = rcp_approx(__fadd_rn(__fadd_rn(u00, u11), S));
    co.A = __fmul_rn(iD, __fmaf_rn(u11, iS, 1.0f));
    co.A2 = __fmul_rn(iD, __fmaf_rn(u00, iS, 1.0f));
    co.Bc = -__fmul_rn(iD, __fmul_rn(u01, iS));
    co.pI = __fmul_rn(__fmul_rn(iD, u0), I);
    co.qI = __fmul_rn(__fmul_rn(iD, u1), I);
    return co;
}

// Alpha-only part shared by the three channels of a pixel: the Coef1 fields
// without the image term; p = u0/D, q = u1/D multiply I_c per channel.  Bn is
// -Bc, kept positive (a product, never a sign-flipped NaN: these values travel
// through sentinel-validated streams, see sweep_full.cu).
struct Coef3 {
    float dL, dR, dU, dD, A, A2, Bn, p, q;
};

__device__ __forceinline__ Coef3 pixel_coef3(float a, float aL, float aR, float aU, float aD, float eps,
                                             float omega) {
    Coef3 co;
    co.dL = edge_weight(a, aL, eps, omega);
    co.dR = edge_weight(a, aR, eps, omega);
    co.dU = edge_weight(a, aU, eps, omega);
    co.dD = edge_weight(a, aD, eps, omega);
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(co.dL, co.dR), co.dU), co.dD);
    const float u0 = a, u1 = __fsub_rn(1.0f, a);
    const float u00 = __fmul_rn(u0, u0), u11 = __fmul_rn(u1, u1), u01 = __fmul_rn(u0, u1);
    const float iS = rcp_approx(S);
    const float iD = rcp_approx(__fadd_rn(__fadd_rn(u00, u11), S));
    co.A = __fmul_rn(iD, __fmaf_rn(u11, iS, 1.0f));
    co.A2 = __fmul_rn(iD, __fmaf_rn(u00, iS, 1.0f));
    co.Bn = __fmul_rn(iD, __fmul_rn(u01, iS));
    co.p = __fmul_rn(iD, u0);
    co.q = __fmul_rn(iD, u1);
    return co;
}

// (x, y) = (F_c, B_c) of the four neighbours; returns the new (F_c, B_c).
__device__ __forceinline__ float2 pixel_apply1(const Coef1& co, float2 L, float2 R, float2 U, float2 D) {
    float SF = __fmul_rn(co.dL, L.x);
    float SB = __fmul_rn(co.dL, L.y);
    SF = __fmaf_rn(co.dD, D.x, SF);
    SB = __fmaf_rn(co.dD, D.y, SB);
    SF = __fmaf_rn(co.dR, R.x, SF);
    SB = __fmaf_rn(co.dR, R.y, SB);
    SF = __fmaf_rn(co.dU, U.x, SF);
    SB = __fmaf_rn(co.dU, U.y, SB);
    return make_float2(__saturatef(__fmaf_rn(co.A, SF, __fmaf_rn(co.Bc, SB, co.pI))),
                       __saturatef(__fmaf_rn(co.A2, SB, __fmaf_rn(co.Bc, SF, co.qI))));
}

// ---- packed (F, B) form: Blackwell's fp32x2 FMA ------------------------------
// Every operation of pixel_coef1_dl / pixel_apply1 is mirrored in (F, B) and
// (u0, u1), so the pairs map onto sm_100's packed fp32 instructions (FFMA2 /
// FMUL2 / FADD2: two IEEE fp32 results per issue slot, with free operand
// broadcast, swap, negation and abs).  Each lane of a pair computes exactly
// the scalar operation of the unpacked form, so results are bitwise equal to
// pixel_coef1_dl + pixel_apply1 (the kernels' cross-check relies on it).  The
// clamp is the one step without a packed form (no .sat on FFMA2): a separate
// saturate per half.  The pre-clamp value is never -0 (A*SF >= +0 and the
// inner term >= +0, see pixel_coef1), so saturate(x) equals FFMA.SAT's.
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 upk2(f32x2 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ f32x2 pk2(float2 v) { return pk2(v.x, v.y); }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// bilerp of two planes at once (same taps): bitwise equal to two bilerp calls.
__device__ __forceinline__ float2 bilerp2(float2 a, float2 b, float2 c, float2 d, float tx, float ty) {
    const f32x2 tx2 = pk2(tx, tx);
    const f32x2 top = fma2(tx2, add2(pk2(b), pk2(-a.x, -a.y)), pk2(a));
    const f32x2 bot = fma2(tx2, add2(pk2(d), pk2(-c.x, -c.y)), pk2(c));
    const float2 tp = upk2(top);
    const float2 r = upk2(fma2(pk2(ty, ty), add2(bot, pk2(-tp.x, -tp.y)), top));
    return make_float2(__saturatef(r.x), __saturatef(r.y));
}

// Coef1 with (A, A2) and (pI, qI) as pairs and Bn = -Bc (negated for free as
// a broadcast operand).
struct CoefP {
    float dL, dR, dU, dD, Bn;
    float2 AA, PQ;
};

__device__ __forceinline__ CoefP pixel_coefp_dl(float a, float dL, float aR, float aU, float aD, float I, float eps,
                                                float omega) {
    CoefP co;
    co.dL = dL;
    {  // (dR, dU) = eps + omega |a - (aR, aU)|
        const float2 df = upk2(add2(pk2(a, a), pk2(-aR, -aU)));
        const float2 d = upk2(fma2(pk2(omega, omega), pk2(fabsf(df.x), fabsf(df.y)), pk2(eps, eps)));
        co.dR = d.x;
        co.dU = d.y;
    }
    co.dD = edge_weight(a, aD, eps, omega);
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(co.dL, co.dR), co.dU), co.dD);
    const float u1 = __fsub_rn(1.0f, a);
    const f32x2 u = pk2(a, u1);
    const float2 uu = upk2(mul2(u, u));  // (u00, u11)
    const float u01 = __fmul_rn(a, u1);
    const float iS = rcp_approx(S);
    const float iD = rcp_approx(__fadd_rn(__fadd_rn(uu.x, uu.y), S));
    const f32x2 iD2 = pk2(iD, iD);
    co.AA = upk2(mul2(iD2, fma2(pk2(uu.y, uu.x), pk2(iS, iS), pk2(1.0f, 1.0f))));
    co.Bn = __fmul_rn(iD, __fmul_rn(u01, iS));
    co.PQ = upk2(mul2(mul2(iD2, u), pk2(I, I)));
    return co;
}

__device__ __forceinline__ float2 pixel_applyp(const CoefP& co, float2 L, float2 R, float2 U, float2 D) {
    f32x2 s = mul2(pk2(co.dL, co.dL), pk2(L));
    s = fma2(pk2(co.dD, co.dD), pk2(D), s);
    s = fma2(pk2(co.dR, co.dR), pk2(R), s);
    s = fma2(pk2(co.dU, co.dU), pk2(U), s);
    const float2 sv = upk2(s);
    const f32x2 t = fma2(pk2(-co.Bn, -co.Bn), pk2(sv.y, sv.x), pk2(co.PQ));
    const float2 r = upk2(fma2(pk2(co.AA), s, t));
    return make_float2(__saturatef(r.x), __saturatef(r.y));
}

// ---- rank-one form (the K3 default) -----------------------------------------
// The matrix is M = S I + u u^T (multilevel.hpp:37-43: a00 = u0^2 + S,
// a01 = u0 u1, a11 = u1^2 + S), so by Sherman-Morrison
//   M^-1 = (I - u u^T / D) / S,   D = |u|^2 + S,
// and with b = I_c u + (SF_c, SB_c), Fbar = SF_c / S, Bbar = SB_c / S:
//   (F_c, B_c) = (Fbar, Bbar) + (u0, u1) / D * (I_c - u0 Fbar - u1 Bbar).
// The same solution as the reference's adj(M) b / det(M) (det = S D), with no
// cancellation beyond the data's own: Fbar is a convex combination of the
// neighbours, the residual I_c - u.(Fbar, Bbar) is bounded by 1 and its
// rounding error is scaled by u0 / D <= 1.  Per pixel: 11 alpha-only
// operations + 2 reciprocals (edge weights, S, D, u/D) and 11 per channel
// (the weighted sums, the residual and the update); the old A/A2/Bc form
// needs ~22 + 8.  Every operation is mirrored in (F, B) / (u0, u1) or is a
// commutative sum of the two halves, so complementing alpha swaps F and B
// bitwise (test_multilevel.cpp:167-180).
struct CoefR {
    float dL, dR, dU, dD, iS, I;
    f32x2 u;   // (a, 1 - a)
    f32x2 pq;  // u / D
};

__device__ __forceinline__ CoefR pixel_coefr_dl(float a, float dL, float aR, float aU, float aD, float I, float eps,
                                                float omega) {
    CoefR co;
    co.dL = dL;
    {  // (dR, dU) = eps + omega |a - (aR, aU)|
        const float2 df = upk2(add2(pk2(a, a), pk2(-aR, -aU)));
        const float2 d = upk2(fma2(pk2(omega, omega), pk2(fabsf(df.x), fabsf(df.y)), pk2(eps, eps)));
        co.dR = d.x;
        co.dU = d.y;
    }
    co.dD = edge_weight(a, aD, eps, omega);
    const float S = __fadd_rn(__fadd_rn(__fadd_rn(co.dL, co.dR), co.dU), co.dD);
    co.u = pk2(a, __fsub_rn(1.0f, a));
    const float2 uu = upk2(mul2(co.u, co.u));
    const float Dn = __fadd_rn(__fadd_rn(uu.x, uu.y), S);
    co.iS = rcp_approx(S);
    const float iD = rcp_approx(Dn);
    co.pq = mul2(pk2(iD, iD), co.u);
    co.I = I;
    return co;
}

__device__ __forceinline__ float2 pixel_applyr(const CoefR& co, float2 L, float2 R, float2 U, float2 D) {
    f32x2 s = mul2(pk2(co.dL, co.dL), pk2(L));
    s = fma2(pk2(co.dD, co.dD), pk2(D), s);
    s = fma2(pk2(co.dR, co.dR), pk2(R), s);
    s = fma2(pk2(co.dU, co.dU), pk2(U), s);
    const f32x2 m = mul2(pk2(co.iS, co.iS), s);  // (Fbar, Bbar)
    const float2 t = upk2(mul2(co.u, m));  // (u0 Fbar, u1 Bbar)
    const float r = __fsub_rn(co.I, __fadd_rn(t.x, t.y));
    // the update as two scalar FFMA.SAT (the same IEEE fma per half as an
    // FFMA2, with the clamp folded in)
    const float2 pq = upk2(co.pq), mv = upk2(m);
    return make_float2(__saturatef(__fmaf_rn(pq.x, r, mv.x)), __saturatef(__fmaf_rn(pq.y, r, mv.y)));
}

// Neighbour-dependent part.  Values from this lane's previous step (L, D)
// enter first, shuffled ones (R, U) last, to keep the recurrence short.
__device__ __forceinline__ void pixel_apply(const Coef& co, const float* L, const float* R, const float* U,
                                            const float* D, float* out) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float SF = __fmul_rn(co.dL, L[c]);
        float SB = __fmul_rn(co.dL, L[3 + c]);
        SF = __fmaf_rn(co.dD, D[c], SF);
        SB = __fmaf_rn(co.dD, D[3 + c], SB);
        SF = __fmaf_rn(co.dR, R[c], SF);
        SB = __fmaf_rn(co.dR, R[3 + c], SB);
        SF = __fmaf_rn(co.dU, U[c], SF);
        SB = __fmaf_rn(co.dU, U[3 + c], SB);
        out[c] = __saturatef(__fmaf_rn(co.A, SF, __fmaf_rn(co.Bc, SB, co.pI[c])));
        out[3 + c] = __saturatef(__fmaf_rn(co.A2, SB, __fmaf_rn(co.Bc, SF, co.qI[c])));
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
