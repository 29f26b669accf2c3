// Microbenchmark (dev tool): gather 128 random 256-B rows per block into a
// 2-stage 128B-swizzled smem ring, the sparse-prefill producer's job.
//   mode 0: 96 threads, cp.async 16 B + wait_group + proxy fence + arrive (shipped)
//   mode 1: one warp, 32 lanes each issue tile::gather4 TMA ops (4 rows x 128 B)
// A consumer warp waits each stage and releases it.  Reports GB/s of gathered rows.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_16391_b200/csrc scripts/micro/gather_bench.cu -o /tmp/gb -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"

using namespace kscd;
using namespace kscd::sm100;

constexpr int kRows = 128, kTile = kRows * 256, kHalf = 16384;

KSCD_DEV void gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

template <int MODE_, int NPROD = 96>
__global__ void __launch_bounds__(NPROD + 32, 1) gather_kernel_t(const __grid_constant__ CUtensorMap tm, const __nv_bfloat16* k,
                                                        const int* pos_all, int nblocks, int npos, float* sink) {
  constexpr int MODE = MODE_;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * 2 * kTile + 65536);   // full[2], empty[2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars[s], (MODE == 0 || MODE == 4) ? NPROD : 1);
      mbar_init(&bars[2 + s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int* pos0 = pos_all + (((size_t)blockIdx.x * 7919 % (npos - nblocks * kRows)) & ~(size_t)3);
  if (warp == NPROD / 32) {
    float acc = 0.f;
    for (int j = 0; j < nblocks; ++j) {
      const int st = j & 1;
      mbar_wait(&bars[st], (j >> 1) & 1);
      acc += reinterpret_cast<float*>(smem + st * 2 * kTile)[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[2 + st]);
    }
    if (lane == 0) sink[blockIdx.x] = acc;
    return;
  }
  for (int j = 0; j < nblocks; ++j) {
    const int st = j & 1;
    if (j >= 2) mbar_wait(&bars[2 + st], ((j >> 1) - 1) & 1);
    const int* pos = pos0 + j * kRows;
    uint8_t* kd = smem + st * 2 * kTile;      // K then V (same rows: stands in for both)
    if (MODE == 4) {
      const uint32_t dst0 = smem_u32(kd);
      for (int rep = 0; rep < 2; ++rep)
        for (int c = threadIdx.x; c < kRows * 16; c += NPROD) {
          const int r = c >> 4, ch = c & 15;
          const int p = __ldg(pos + r);
          const uint32_t off = rep * kTile + (ch >> 3) * kHalf + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
          cp_async16_zfill(dst0 + off, k + (int64_t)p * 128 + ch * 8, true);
        }
      cp_async_mbar_arrive(&bars[st]);     // arrives when this thread's copies land; no blocking wait
    } else if (MODE == 0) {
      const uint32_t dst0 = smem_u32(kd);
      // positions staged in shared memory first (as the prefill producer does)
      int* spos = reinterpret_cast<int*>(smem + 2 * 2 * kTile + 65536 + 64);
      for (int r = threadIdx.x; r < kRows; r += NPROD) spos[r] = __ldg(pos + r);
      asm volatile("bar.sync 1, %0;\n" ::"r"(NPROD));
      for (int rep = 0; rep < 2; ++rep) {
        for (int c = threadIdx.x; c < kRows * 16; c += NPROD) {
          const int r = c >> 4, ch = c & 15;
          const int p = spos[r];
          const uint32_t off = rep * kTile + (ch >> 3) * kHalf + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
          cp_async16_zfill(dst0 + off, k + (int64_t)p * 128 + ch * 8, true);
        }
        cp_async_commit();
      }
      cp_async_wait<0>();
      fence_proxy_async_smem();
      mbar_arrive(&bars[st]);
    } else if (warp == 0 && MODE == 1) {
      if (lane == 0) mbar_expect_tx(&bars[st], 2 * kTile);
      __syncwarp();
      // 2 (K,V) x 2 halves x 32 row groups = 128 gather4 ops; 4 per lane
      for (int op = lane; op < 128; op += 32) {
        const int rep = op >> 6, hf = (op >> 5) & 1, grp = op & 31;
        const int4 p = __ldg(reinterpret_cast<const int4*>(pos + grp * 4));
        gather4(kd + rep * kTile + hf * kHalf + grp * 512, &tm, &bars[st], hf * 64, p.x, p.y, p.z, p.w);
      }
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int nrows = argc > 3 ? atoi(argv[3]) : 131072;   // 131072 rows = 32 MB (L2-resident); 16M rows = 4 GB (HBM)
  const int nblocks = argc > 1 ? atoi(argv[1]) : 50;
  const int grid = argc > 2 ? atoi(argv[2]) : 148;
  const int npos = 200000;
  __nv_bfloat16* k;
  int* pos;
  float* sink;
  cudaMalloc(&k, (size_t)nrows * 256);
  cudaMemset(k, 0, (size_t)nrows * 256);
  std::vector<int> hp(npos);
  srand(1);
  for (int i = 0; i < npos; i += kRows) {     // sorted random selections per block, like Top-k lists
    std::vector<int> blk(kRows);
    for (int r = 0; r < kRows; ++r) blk[r] = (int)(((long long)rand() * 32768 + rand()) % nrows);
    std::sort(blk.begin(), blk.end());
    for (int r = 0; r < kRows && i + r < npos; ++r) hp[i + r] = blk[r];
  }
  cudaMalloc(&pos, npos * 4);
  cudaMemcpy(pos, hp.data(), npos * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, grid * 4);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {128, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = ((EncodeFn)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) { printf("encode failed %d\n", (int)rc); return 1; }
  const int smem = 2 * 2 * kTile + 64 + 1024 + 65536 + 1024;
  cudaFuncSetAttribute(gather_kernel_t<0, 96>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel_t<1, 96>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel_t<0, 192>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel_t<0, 288>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gather_kernel_t<4, 96>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = (argc > 5 ? atoi(argv[5]) : 0); mode < (argc > 4 ? atoi(argv[4]) : 2); ++mode) {
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(a);
      if (mode == 0) gather_kernel_t<0, 96><<<grid, 128, smem>>>(tm, k, pos, nblocks, npos, sink);
      else if (mode == 1) gather_kernel_t<1, 96><<<grid, 128, smem>>>(tm, k, pos, nblocks, npos, sink);
      else if (mode == 2) gather_kernel_t<0, 192><<<grid, 224, smem>>>(tm, k, pos, nblocks, npos, sink);
      else if (mode == 3) gather_kernel_t<0, 288><<<grid, 320, smem>>>(tm, k, pos, nblocks, npos, sink);
      else gather_kernel_t<4, 96><<<grid, 128, smem>>>(tm, k, pos, nblocks, npos, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      double bytes = (double)grid * nblocks * 2 * kTile;
      printf("mode %d grid %d blocks %d: %.3f ms  %.0f GB/s  per-SM %.1f B/clk@1.9GHz  %s\n", mode, grid, nblocks, ms,
             bytes / ms / 1e6, bytes / ms / 1e6 / grid / 1.9, cudaGetErrorString(e));
    }
  }
  return 0;
}
