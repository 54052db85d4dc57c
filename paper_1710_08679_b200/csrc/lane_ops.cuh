// lane_ops.cuh — arithmetic on the per-thread "lane vector" of load cases.
//
// A thread owns CPT consecutive load cases (columns) of one element. For fp32
// CPT = 2 and every operation is one packed sm_100 instruction
// (FFMA2 / FADD2 / FMUL2: __ffma2_rn & co.), which doubles FP32 throughput
// over scalar 3-register FFMA; for fp64 CPT = 1 (DFMA). Coefficients that are
// per element (gradients, scaled Lame pairs) are splatted once.
#pragma once
#include <cuda_runtime.h>

namespace tsg {

template <typename V> struct LaneOps;

template <> struct LaneOps<float2> {
  using S = float;
  static constexpr int kCols = 2;
  __device__ __forceinline__ static float2 zero() { return make_float2(0.f, 0.f); }
  __device__ __forceinline__ static float2 splat(float s) { return make_float2(s, s); }
  __device__ __forceinline__ static float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
  __device__ __forceinline__ static float2 sub(float2 a, float2 b) {
    return __ffma2_rn(b, make_float2(-1.f, -1.f), a);
  }
  __device__ __forceinline__ static float2 mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
  __device__ __forceinline__ static float2 fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
  // only as an FFMA2 operand: the sign folds into the instruction (no extra op)
  __device__ __forceinline__ static float2 neg(float2 a) { return make_float2(-a.x, -a.y); }
  // c - a*b
  __device__ __forceinline__ static float2 fnma(float2 a, float2 b, float2 c) {
    return __ffma2_rn(make_float2(-a.x, -a.y), b, c);
  }
};

// Scalar lanes round exactly like one lane of the packed ops (explicit _rn
// intrinsics: no FMA contraction of a separate mul + add), so a case's result
// does not depend on whether the batch width selected packed or scalar lanes.
template <> struct LaneOps<float> {
  using S = float;
  static constexpr int kCols = 1;
  __device__ __forceinline__ static float zero() { return 0.f; }
  __device__ __forceinline__ static float splat(float s) { return s; }
  __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static float sub(float a, float b) { return __fmaf_rn(b, -1.f, a); }
  __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
  __device__ __forceinline__ static float neg(float a) { return -a; }
  __device__ __forceinline__ static float fnma(float a, float b, float c) { return __fmaf_rn(-a, b, c); }
};

template <> struct LaneOps<double> {
  using S = double;
  static constexpr int kCols = 1;
  __device__ __forceinline__ static double zero() { return 0.0; }
  __device__ __forceinline__ static double splat(double s) { return s; }
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
  __device__ __forceinline__ static double neg(double a) { return -a; }
  __device__ __forceinline__ static double fnma(double a, double b, double c) { return ::fma(-a, b, c); }
};

// ---- lane-vector global memory access ----------------------------------------
__device__ __forceinline__ float2 ld_lane(const float2* p) { return __ldg(p); }
__device__ __forceinline__ float ld_lane(const float* p) { return __ldg(p); }
__device__ __forceinline__ double ld_lane(const double* p) { return __ldg(p); }

// fire-and-forget atomic accumulation (REDG); fp32 pairs use the sm_90+ vector form
__device__ __forceinline__ void red_lane(float2* p, float2 v) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void red_lane(float* p, float v) { atomicAdd(p, v); }
__device__ __forceinline__ void red_lane(double* p, double v) { atomicAdd(p, v); }

}  // namespace tsg
