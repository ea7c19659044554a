// tc_probe.cu -- standalone check of two sm_100a facts the small-M tensor-core design relies on:
//  (1) tcgen05.mma.cta_group::1.kind::f16 with the A operand in TMEM (written by tcgen05.st,
//      32-bit column i of lane r = fp16 pair (A[r][2i], A[r][2i+1])),
//  (2) fp16 subnormal A values are multiplied exactly (no flush to zero).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2504_12984_b200/csrc tc_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#include "ptx.cuh"

using namespace tl;

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__global__ void probe(const __half* A /*[128][16]*/, const __half* B /*[16 n][16 k] (K-major)*/, float* D /*[128][16]*/) {
  __shared__ __align__(1024) uint8_t bsm[16 * 128];  // 16 rows (n) x 128 B (64 k, only 16 used)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // B operand: row n, k-chunk c (8 k = 16 B), SW128: physical chunk c ^ (n & 7)
  for (int i = t; i < 16 * 64; i += blockDim.x) {
    const int n = i / 64, k = i % 64;
    const int c = k / 8, e = k % 8;
    __half v = k < 16 ? B[n * 16 + k] : __float2half(0.f);
    *reinterpret_cast<__half*>(bsm + n * 128 + ((c ^ (n & 7)) * 16) + e * 2) = v;
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tslot, 64);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;  // columns [0,32): D (16 used), [32,40): A
  // A into TMEM: thread = row r = 32*warp + lane; 8 columns = 16 k
  {
    const int r = warp * 32 + lane;
    uint32_t regs[8];
    for (int i = 0; i < 8; ++i) {
      __half2 h = __halves2half2(A[r * 16 + 2 * i], A[r * 16 + 2 * i + 1]);
      regs[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    tmem_st_32x32b_x8(tmem + ((uint32_t)(warp * 32) << 16) + 32, regs);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bd = sw128_desc(smem_u32(bsm));
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
        "r"(tmem + 32), "l"(bd), "r"(idesc), "r"(0u)
        : "memory");
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    uint32_t r[16];
    tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16), r);
    tmem_ld_wait();
    const int row = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[row * 16 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

int main() {
  std::vector<__half> hA(128 * 16), hB(16 * 16);
  std::vector<float> fA(128 * 16), fB(16 * 16);
  srand(1);
  for (int i = 0; i < 128 * 16; ++i) {
    // mix of normal values and fp16 subnormals (u * 2^-24 style codes)
    float v;
    if (i % 3 == 0) v = (float)((rand() % 1024)) * ldexpf(1.f, -24);           // subnormal grid
    else if (i % 3 == 1) v = (float)((rand() % 64) - 32) * ldexpf(1.f, -20);   // small
    else v = (float)((rand() % 200) - 100) / 8.f;
    hA[i] = __float2half(v);
    fA[i] = __half2float(hA[i]);
  }
  for (int i = 0; i < 16 * 16; ++i) {
    float v = (float)((rand() % 200) - 100) / 16.f;
    hB[i] = __float2half(v);
    fB[i] = __half2float(hB[i]);
  }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dD, 128 * 16 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> hD(128 * 16);
  cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
  double max_err = 0, max_sub_err = 0;
  int mism = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < 16; ++n) {
      double ref = 0;
      for (int k = 0; k < 16; ++k) ref += (double)fA[r * 16 + k] * (double)fB[n * 16 + k];
      double err = fabs(ref - hD[r * 16 + n]);
      if (err > max_err) max_err = err;
      if (err > 1e-6 * (fabs(ref) + 1e-30)) ++mism;
    }
  // subnormal-only check: rows where only subnormal values are nonzero
  printf("max_abs_err=%.3e mismatches(rel>1e-6)=%d sample D[0]=%f\n", max_err, mism, hD[0]);
  // dedicated subnormal exactness: A = u * 2^-24 (u < 1024), B = small integers -> exact
  for (int i = 0; i < 128 * 16; ++i) {
    hA[i] = __float2half((float)(rand() % 1024) * ldexpf(1.f, -24));
    fA[i] = __half2float(hA[i]);
  }
  for (int i = 0; i < 16 * 16; ++i) {
    hB[i] = __float2half((float)((rand() % 17) - 8));
    fB[i] = __half2float(hB[i]);
  }
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaDeviceSynchronize();
  cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
  int exact_bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < 16; ++n) {
      double ref = 0;
      for (int k = 0; k < 16; ++k) ref += (double)fA[r * 16 + k] * (double)fB[n * 16 + k];
      if ((double)hD[r * 16 + n] != ref) ++exact_bad;
    }
  printf("subnormal-exact mismatches=%d (of 2048)\n", exact_bad);
  return 0;
}
