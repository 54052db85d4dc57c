// Memory-path microbenchmark for the EBE sweep (r = 16 fp32, config-2 sized
// tet10 box): gather 10 node rows (192 B each) per element, trivial compute,
// scatter-add 10 node rows. Variants:
//   A: cp.async 8 B per (thread, dof) + red.v2 per (thread, dof)        [current production pattern]
//   B: cp.async 16 B per node chunk + red.v4 per node chunk (8 thr/elem)
//   C: TMA bulk copy 192 B per node (mbarrier) + bulk reduce-add 192 B per node from smem
//   D: plain ld.global.v2 (no staging) + red.v2
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)
constexpr int R = 16, NPE = 10, ROW = 3 * R;  // floats per node row

__device__ __forceinline__ void cpa(void* s, const void* g, int bytes) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void red2(float* p, float2 v) { asm volatile("red.global.add.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory"); }
__device__ __forceinline__ void red4(float* p, float4 v) { asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory"); }

// A: 8 threads per element, each 2 cases x 30 dofs
__global__ void __launch_bounds__(128, 4) kA(const int* conn, int E, const float* u, float* f) {
  extern __shared__ __align__(16) float2 bufA[]; auto buf = reinterpret_cast<float2 (*)[30][128]>(bufA);
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8, G = gridDim.x * 16;
  int e = blockIdx.x * 16 + grp, s = 0;
  auto issue = [&](int ee, int st) {
    if (ee < E) for (int a = 0; a < NPE; ++a) { int n = __ldg(conn + ee * NPE + a);
      for (int c = 0; c < 3; ++c) cpa(&buf[st][a * 3 + c][threadIdx.x], u + (size_t)n * ROW + c * R + 2 * l, 8); }
    asm volatile("cp.async.commit_group;");
  };
  issue(e, 0);
  while (__any_sync(~0u, e < E)) {
    issue(e + G, s ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory"); __syncwarp();
    if (e < E) for (int a = 0; a < NPE; ++a) { int n = __ldg(conn + e * NPE + a);
      for (int c = 0; c < 3; ++c) { float2 v = buf[s][a * 3 + c][threadIdx.x]; v.x *= 1.5f; v.y *= 1.5f; red2(f + (size_t)n * ROW + c * R + 2 * l, v); } }
    __syncwarp(); e += G; s ^= 1;
  }
}
// B: 8 threads per element; node row = 12 x 16 B chunks; 120 chunks / 8 thr = 15 each
__global__ void __launch_bounds__(128, 4) kB(const int* conn, int E, const float* u, float* f) {
  extern __shared__ __align__(16) float4 bufB[]; auto buf = reinterpret_cast<float4 (*)[16][120]>(bufB);
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8, G = gridDim.x * 16;
  int e = blockIdx.x * 16 + grp, s = 0;
  auto issue = [&](int ee, int st) {
    if (ee < E) for (int k = l; k < 120; k += 8) { int a = k / 12, ch = k % 12; int n = __ldg(conn + ee * NPE + a);
      cpa(&buf[st][grp][k], u + (size_t)n * ROW + ch * 4, 16); }
    asm volatile("cp.async.commit_group;");
  };
  issue(e, 0);
  while (__any_sync(~0u, e < E)) {
    issue(e + G, s ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory"); __syncwarp();
    if (e < E) for (int k = l; k < 120; k += 8) { int a = k / 12, ch = k % 12; int n = __ldg(conn + e * NPE + a);
      float4 v = buf[s][grp][k]; v.x *= 1.5f; v.y *= 1.5f; v.z *= 1.5f; v.w *= 1.5f; red4(f + (size_t)n * ROW + ch * 4, v); }
    __syncwarp(); e += G; s ^= 1;
  }
}
// C: TMA bulk. warp = 4 elements per step; lane 0 issues 40 bulk loads (192 B) / 40 bulk reduces.
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) kC(const int* conn, int E, const float* u, float* f) {
  extern __shared__ __align__(128) float sm[];
  constexpr int SLOT = 40 * ROW;  // floats per stage per warp (4 elements x 10 nodes x 48)
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32, grp = lane / 8, l = lane % 8;
  float* ub = sm + w * 4 * SLOT;           // [2 stages][SLOT]
  float* fb = ub + 2 * SLOT;               // [2 stages][SLOT]
  __shared__ __align__(8) uint64_t mbar[WARPS][2];
  if (lane == 0) for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int G = gridDim.x * WARPS * 4;
  int e0 = (blockIdx.x * WARPS + w) * 4;
  auto issue = [&](int eb, int st) {
    if (lane == 0 && eb < E) {
      int ne = min(4, E - eb);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mbar[w][st])), "r"(ne * 10 * ROW * 4) : "memory");
      for (int k = 0; k < ne * 10; ++k) { int n = __ldg(conn + eb * NPE + k);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(ub + st * SLOT + k * ROW)), "l"(u + (size_t)n * ROW), "r"(ROW * 4), "r"(sa(&mbar[w][st])) : "memory"); }
    }
  };
  issue(e0, 0);
  int s = 0; unsigned ph[2] = {0, 0};
  while (e0 < E) {
    issue(e0 + G, s ^ 1);
    { unsigned done = 0; while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(sa(&mbar[w][s])), "r"(ph[s]) : "memory"); }
    ph[s] ^= 1;
    // f stage s is free once the bulk reduces issued two steps ago have read it
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    const int e = e0 + grp;
    if (e < E) for (int q = 0; q < 30; ++q) { float2 v = *reinterpret_cast<float2*>(ub + s * SLOT + (grp * 30 + q) * R + 2 * l);
      v.x *= 1.5f; v.y *= 1.5f; *reinterpret_cast<float2*>(fb + s * SLOT + (grp * 30 + q) * R + 2 * l) = v; }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) { int ne = min(4, E - e0);
      for (int k = 0; k < ne * 10; ++k) { int n = __ldg(conn + e0 * NPE + k);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                     ::"l"(f + (size_t)n * ROW), "r"(sa(fb + s * SLOT + k * ROW)), "r"(ROW * 4) : "memory"); }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
    e0 += G; s ^= 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// D: direct loads to registers
__global__ void __launch_bounds__(128, 8) kD(const int* conn, int E, const float* u, float* f) {
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8;
  for (int e = blockIdx.x * 16 + grp; e < E; e += gridDim.x * 16) {
    float2 v[30]; int n[10];
    for (int a = 0; a < 10; ++a) n[a] = __ldg(conn + e * NPE + a);
    for (int a = 0; a < 10; ++a) for (int c = 0; c < 3; ++c) v[a * 3 + c] = __ldg(reinterpret_cast<const float2*>(u + (size_t)n[a] * ROW + c * R + 2 * l));
    for (int a = 0; a < 10; ++a) for (int c = 0; c < 3; ++c) { float2 x = v[a * 3 + c]; x.x *= 1.5f; x.y *= 1.5f; red2(f + (size_t)n[a] * ROW + c * R + 2 * l, x); }
  }
}


// A1: gather only (cp.async 8 B), sum into one value per element
__global__ void __launch_bounds__(128, 4) kA1(const int* conn, int E, const float* u, float* f) {
  extern __shared__ __align__(16) float2 bufA1[]; auto buf = reinterpret_cast<float2 (*)[30][128]>(bufA1);
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8, G = gridDim.x * 16;
  int e = blockIdx.x * 16 + grp, s = 0; float acc = 0;
  auto issue = [&](int ee, int st) {
    if (ee < E) for (int a = 0; a < NPE; ++a) { int n = __ldg(conn + ee * NPE + a);
      for (int c = 0; c < 3; ++c) cpa(&buf[st][a * 3 + c][threadIdx.x], u + (size_t)n * ROW + c * R + 2 * l, 8); }
    asm volatile("cp.async.commit_group;");
  };
  issue(e, 0);
  while (__any_sync(~0u, e < E)) {
    issue(e + G, s ^ 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory"); __syncwarp();
    if (e < E) for (int q = 0; q < 30; ++q) { float2 v = buf[s][q][threadIdx.x]; acc += v.x + v.y; }
    __syncwarp(); e += G; s ^= 1;
  }
  if (acc == 1.2345f) f[0] = acc;
}
// A2: scatter only, red.v2 ; A3: scatter only, st.global.v2 (racy; traffic reference)
template <bool ATOMIC>
__global__ void __launch_bounds__(128, 8) kS2(const int* conn, int E, const float* u, float* f) {
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8;
  for (int e = blockIdx.x * 16 + grp; e < E; e += gridDim.x * 16) {
    int n[10]; for (int a = 0; a < 10; ++a) n[a] = __ldg(conn + e * NPE + a);
    for (int a = 0; a < 10; ++a) for (int c = 0; c < 3; ++c) { float2 x = make_float2(1.f, 2.f); float* p = f + (size_t)n[a] * ROW + c * R + 2 * l;
      if (ATOMIC) red2(p, x); else *reinterpret_cast<float2*>(p) = x; }
  }
}
// S4: scatter only red.v4 per node chunk (coalesced 192 B rows)
__global__ void __launch_bounds__(128, 8) kS4(const int* conn, int E, const float* u, float* f) {
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8;
  for (int e = blockIdx.x * 16 + grp; e < E; e += gridDim.x * 16) {
    for (int k = l; k < 120; k += 8) { int a = k / 12, ch = k % 12; int n = __ldg(conn + e * NPE + a);
      red4(f + (size_t)n * ROW + ch * 4, make_float4(1.f, 2.f, 3.f, 4.f)); }
  }
}
// S4 into a small (L2-resident) target: node index folded mod NS
__global__ void __launch_bounds__(128, 8) kS4small(const int* conn, int E, const float* u, float* f, int NS) {
  const int grp = threadIdx.x / 8, l = threadIdx.x % 8;
  for (int e = blockIdx.x * 16 + grp; e < E; e += gridDim.x * 16) {
    for (int k = l; k < 120; k += 8) { int a = k / 12, ch = k % 12; int n = __ldg(conn + e * NPE + a) % NS;
      red4(f + (size_t)n * ROW + ch * 4, make_float4(1.f, 2.f, 3.f, 4.f)); }
  }
}
// streaming reference: contiguous red.v4 over f (each row once) and copy u->f
__global__ void kStreamRed(float* f, long n4) { for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) red4(f + 4 * i, make_float4(1.f, 1.f, 1.f, 1.f)); }
__global__ void kCopy(const float4* u, float4* f, long n4) { for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) f[i] = u[i]; }

int main() {
  const int nx = 82, ny = 123, nz = 41, X = 2 * nx + 1, Y = 2 * ny + 1, Z = 2 * nz + 1;
  const long N = (long)X * Y * Z; const int E = 6 * nx * ny * nz;
  std::vector<int> conn((size_t)E * NPE);
  const int perm[6][3] = {{0,1,2},{0,2,1},{1,0,2},{1,2,0},{2,0,1},{2,1,0}};
  const int ed[6][2] = {{0,1},{1,2},{2,0},{0,3},{1,3},{2,3}};
  long e = 0;
  for (int i = 0; i < nx; ++i) for (int j = 0; j < ny; ++j) for (int k = 0; k < nz; ++k)
    for (int t = 0; t < 6; ++t) {
      int v[4][3]; int p[3] = {0, 0, 0};
      for (int d = 0; d < 3; ++d) v[0][d] = 0;
      for (int m = 0; m < 3; ++m) { p[perm[t][m]] = 1; for (int d = 0; d < 3; ++d) v[m + 1][d] = p[d]; }
      int g[10][3];
      for (int a = 0; a < 4; ++a) { g[a][0] = 2 * (i + v[a][0]); g[a][1] = 2 * (j + v[a][1]); g[a][2] = 2 * (k + v[a][2]); }
      for (int q = 0; q < 6; ++q) for (int d = 0; d < 3; ++d) g[4 + q][d] = (g[ed[q][0]][d] + g[ed[q][1]][d]) / 2;
      for (int a = 0; a < 10; ++a) conn[e * NPE + a] = (g[a][0] * Y + g[a][1]) * Z + g[a][2];
      ++e;
    }
  int* dconn; float *u, *f;
  CK(cudaMalloc(&dconn, conn.size() * 4)); CK(cudaMemcpy(dconn, conn.data(), conn.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&u, N * ROW * 4)); CK(cudaMalloc(&f, N * ROW * 4));
  CK(cudaMemset(u, 0, N * ROW * 4)); CK(cudaMemset(f, 0, N * ROW * 4));
  double alg = (double)E * NPE * 4 + 2.0 * N * ROW * 4;
  printf("E=%d N=%ld alg bytes (conn + u + f) = %.3f GB\n", E, N, alg / 1e9);
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto time = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a)); for (int w = 0; w < 10; ++w) launch(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); ms /= 10;
    printf("%-28s %.4f ms  %.0f GB/s alg\n", name, ms, alg / ms / 1e6);
  };
  CK(cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, 61440));
  time("A cp.async8+red.v2", [&] { kA<<<148 * 3, 128, 61440>>>(dconn, E, u, f); });
  CK(cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, 61440));
  time("B cp.async16+red.v4", [&] { kB<<<148 * 3, 128, 61440>>>(dconn, E, u, f); });
  time("D ldg.v2+red.v2", [&] { kD<<<148 * 8, 128>>>(dconn, E, u, f); });
  {
    constexpr int W = 4; size_t sm = W * 4 * 40 * ROW * 4;
    CK(cudaFuncSetAttribute(kC<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    time("C tma bulk W4", [&] { kC<W><<<148, W * 32, sm>>>(dconn, E, u, f); });
  }
  {
    constexpr int W = 2; size_t sm = W * 4 * 40 * ROW * 4;
    CK(cudaFuncSetAttribute(kC<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    time("C tma bulk W2 x2cta", [&] { kC<W><<<296, W * 32, sm>>>(dconn, E, u, f); });
  }

  CK(cudaFuncSetAttribute(kA1, cudaFuncAttributeMaxDynamicSharedMemorySize, 61440));
  time("A1 gather only cp.async8", [&] { kA1<<<148 * 3, 128, 61440>>>(dconn, E, u, f); });
  time("S2 scatter only red.v2", [&] { kS2<true><<<148 * 8, 128>>>(dconn, E, u, f); });
  time("S2 scatter only st.v2", [&] { kS2<false><<<148 * 8, 128>>>(dconn, E, u, f); });
  time("S4 scatter only red.v4", [&] { kS4<<<148 * 8, 128>>>(dconn, E, u, f); });
  time("S4 red.v4 L2-resident 24MB", [&] { kS4small<<<148 * 8, 128>>>(dconn, E, u, f, 131072); });
  time("stream red.v4 over f", [&] { kStreamRed<<<148 * 8, 256>>>(f, N * ROW / 4); });
  time("copy u->f", [&] { kCopy<<<148 * 8, 256>>>((const float4*)u, (float4*)f, N * ROW / 4); });
  CK(cudaGetLastError());
  return 0;
}
