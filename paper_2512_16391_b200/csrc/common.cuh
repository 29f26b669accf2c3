// Shared device helpers for the Kascade B200 engine (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "kascade_b200 is written for sm_100a (B200) only"
#endif

#define KSCD_DEV __device__ __forceinline__

namespace kscd {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kHeadDim = 128;           // the engine's only head dim (256-B bf16 rows)
constexpr int kRowBytes = kHeadDim * 2;
constexpr int kChunksPerRow = kRowBytes / 16;   // 16 x 16-byte chunks per K/V row

// ---------------------------------------------------------------- memory ops
KSCD_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte global->shared async copy (LDGSTS), L1 bypassed: K/V rows are
// streamed exactly once per CTA.
KSCD_DEV void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
KSCD_DEV void cp_async16_zfill(uint32_t dst, const void* src, bool valid) {
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
KSCD_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
KSCD_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// XOR swizzle of the 16-byte chunk index inside a 256-byte row: the 8 rows
// an ldmatrix 8x8 tile touches land in 8 distinct bank groups.
KSCD_DEV int swz(int row, int chunk) { return chunk ^ (row & 7); }

KSCD_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
KSCD_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D (fp32).  Used only for the
// decode GEMVs (G <= 16 query heads x 16 keys), where the tensor pipe is
// <5% busy and HBM is the bound; prefill uses tcgen05.
KSCD_DEV void mma_bf16_16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                             uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

KSCD_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

KSCD_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// exp2 of a pair on the FMA pipe (Cody-Waite split + degree-6 minimax of
// 2^f on [-0.5, 0.5], max rel. error 9e-8 in fp32 -- on par with MUFU.EX2).
// Softmax loops send a fixed share of their exponentials here so the MUFU
// unit (16/clk/SM on B200) stops being the only exp engine.  Inputs below
// -126 (incl. -inf for masked keys) return exact zeros.
KSCD_DEV float2 exp2_poly2(float2 x) {
  const float2 xc = make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f));
  const float2 t = __fadd2_rn(xc, make_float2(12582912.f, 12582912.f));      // round to integer
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(n, make_float2(-1.f, -1.f), xc);               // f = x - n
  float2 p = make_float2(1.4990878116805106e-04f, 1.4990878116805106e-04f);
  p = __ffma2_rn(p, f, make_float2(1.339308568276465e-03f, 1.339308568276465e-03f));
  p = __ffma2_rn(p, f, make_float2(9.61967371404171e-03f, 9.61967371404171e-03f));
  p = __ffma2_rn(p, f, make_float2(5.5503472685813904e-02f, 5.5503472685813904e-02f));
  p = __ffma2_rn(p, f, make_float2(2.402263730764389e-01f, 2.402263730764389e-01f));
  p = __ffma2_rn(p, f, make_float2(6.931471824645996e-01f, 6.931471824645996e-01f));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  // 2^n: the low bits of t hold n, so t_bits << 23 == n << 23 (mod 2^32)
  const float rx = __int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23));
  const float ry = __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23));
  return make_float2(x.x < -126.f ? 0.f : rx, x.y < -126.f ? 0.f : ry);
}

// exp2 of a pair: FMA-pipe polynomial for pair indices with (pair & 7) <
// kPolyPairsPer8, MUFU for the rest.  `pair` is a compile-time constant
// inside the fully unrolled softmax loops, so the split costs nothing.
// Measured on B200 (128K prefill): 3/8 polynomial made the dense / LSE /
// pass-B kernels 10-16% SLOWER (extra issue slots + register spills), so the
// split is off; the kernels are issue/latency bound, not MUFU bound.
#ifdef KSCD_POLY
constexpr int kPolyPairsPer8 = KSCD_POLY;
#else
constexpr int kPolyPairsPer8 = 0;
#endif
// Share of the exponentials of the two anchor passes (row sums of pass A,
// column sums of pass B) that go to the FMA-pipe polynomial.  Measured on
// B200 (same box, A/B alternated): at 32K, 1/8-2/8 cut pass A by 6-13%
// (pass B within noise); at 128K every split is within +-1% of MUFU-only --
// the long launches run under sw_power_cap, so offloaded exponentials buy
// no clock cycles.  1/8 is kept as the smallest deviation from MUFU.EX2.
#ifndef KSCD_PB_POLY
#define KSCD_PB_POLY 1      // pass B column sums: polynomial pairs per 8
#endif
#ifndef KSCD_LSE_POLY
#define KSCD_LSE_POLY 1     // pass A row sums: polynomial pairs per 8
#endif
KSCD_DEV float2 exp2_pair(float2 x, int pair) {
  if ((pair & 7) < kPolyPairsPer8) return exp2_poly2(x);
  return make_float2(fast_exp2(x.x), fast_exp2(x.y));
}

// exp2 of a pair on the FMA pipe for inputs that never need an exact zero
// (anchor pass A row sums, pass B column sums): Cody-Waite split + degree-5
// minimax of 2^f on [-0.5, 0.5] (max rel. error 2.3e-7 in fp32, the same
// class as MUFU.EX2's 2^-22).  Inputs below -126 (incl. -inf) return
// 2^-126 instead of 0 -- harmless inside a sum of terms >= 2^-126 * count.
KSCD_DEV float2 exp2_poly5(float2 x) {
  const float2 xc = make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f));
  const float2 t = __fadd2_rn(xc, make_float2(12582912.f, 12582912.f));      // round to integer
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(n, make_float2(-1.f, -1.f), xc);               // f = x - n
  float2 p = make_float2(0.00132764654699713f, 0.00132764654699713f);
  p = __ffma2_rn(p, f, make_float2(0.009675540961325169f, 0.009675540961325169f));
  p = __ffma2_rn(p, f, make_float2(0.05550713464617729f, 0.05550713464617729f));
  p = __ffma2_rn(p, f, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = __ffma2_rn(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// exp2 of a pair for sums: FMA-pipe polynomial for pair indices with
// (pair & 7) < POLY, MUFU for the rest (POLY is a compile-time split).
template <int POLY>
KSCD_DEV float2 exp2_pair_sum(float2 x, int pair) {
  if ((pair & 7) < POLY) return exp2_poly5(x);
  return make_float2(fast_exp2(x.x), fast_exp2(x.y));
}

KSCD_DEV float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// Max of N register values as 8 independent FMNMX3 chains and a short
// combine (a single running max is a 64-deep dependent chain at N = 128).
template <int N>
KSCD_DEV float max_tree(const float* s) {
  static_assert(N % 16 == 0, "N must be a multiple of 16");
  float m[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) m[k] = fmaxf(s[2 * k], s[2 * k + 1]);
#pragma unroll
  for (int c = 16; c < N; c += 16)
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = fmaxf(m[k], fmaxf(s[c + 2 * k], s[c + 2 * k + 1]));
  const float a = fmaxf(m[0], fmaxf(m[1], m[2]));
  const float b = fmaxf(m[3], fmaxf(m[4], m[5]));
  return fmaxf(fmaxf(a, b), fmaxf(m[6], m[7]));
}

template <typename T>
KSCD_DEV T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <typename T>
KSCD_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// k_budget (tiles.py:81-89) on the device: floor of the fp64 product,
// clamped below by k_min and above by n (the host's kscd_k_budget).
KSCD_DEV int k_budget_dev(double fraction, int k_min, int n) {
  long long kk = (long long)floor(fraction * (double)n);
  kk = kk < k_min ? k_min : kk;
  return (int)(kk > n ? n : kk);
}

}  // namespace kscd
