// Layout self-test of the tcgen05 building blocks used by the NN and SKUT
// kernels: one 128 x N x K MMA per case, compared against a host reference
// by tests/test_gpu_tc.py.  Cases:
//   0 bf16, A smem K-major, B smem K-major
//   1 bf16, A from TMEM,    B smem K-major
//   2 bf16, A smem K-major, B smem MN-major
//   3 i8,   A smem K-major, B loaded by TMA (3-D chunk-major map)
//   4 i8,   A smem K-major, B smem K-major (manual load)
//   5 bf16, A smem K-major, B smem MN-major with the core matrices tiled
//     k-group-fastest: (k, n) at (n/8)*(K*16) + (k/8)*128 + (k%8)*16 +
//     (n%8)*2 (LBO = 128, SBO = K*16) -- skut_tc4 reads its key buffer,
//     written K-major for S = Q'K^T, as this MN-major B of P.a
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"
#include "tc_common.cuh"

namespace tav2 {

using namespace tc;

__global__ void __launch_bounds__(128) tc_selftest_kernel(int which, const uint8_t* A, const uint8_t* B,
                                                          void* D, int N, int K,
                                                          const __grid_constant__ CUtensorMap mapB) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool i8 = which == 3 || which == 4;
  const int esz = i8 ? 1 : 2;
  const int kbytes = K * esz;           // bytes per row
  const int nchunk = kbytes / 16;       // 16-byte K chunks
  uint8_t* As = sm;                     // 128 rows
  uint8_t* Bs = sm + 128 * kbytes;      // N rows (or MN-major K x N)
  // ---- A: K-major chunk slabs ----
  for (int c = 0; c < nchunk; ++c) {
    *reinterpret_cast<int4*>(As + c * 128 * 16 + tid * 16) =
        *reinterpret_cast<const int4*>(A + (size_t)tid * kbytes + c * 16);
  }
  // ---- B ----
  if (which == 5) {  // MN-major, k-groups fastest: global [K][N] bf16
    for (int e = tid; e < K * (N / 8); e += 128) {
      int k = e / (N / 8), g = e % (N / 8);
      *reinterpret_cast<int4*>(Bs + g * (K * 16) + (k / 8) * 128 + (k % 8) * 16) =
          *reinterpret_cast<const int4*>(B + ((size_t)k * N + g * 8) * 2);
    }
  } else if (which == 2) {  // MN-major: global [K][N] bf16
    const int lbo = (N / 8) * 128;
    for (int e = tid; e < K * (N / 8); e += 128) {
      int k = e / (N / 8), g = e % (N / 8);
      *reinterpret_cast<int4*>(Bs + (k / 8) * lbo + g * 128 + (k % 8) * 16) =
          *reinterpret_cast<const int4*>(B + ((size_t)k * N + g * 8) * 2);
    }
  } else if (which != 3) {
    for (int e = tid; e < N * nchunk; e += 128) {
      int n = e / nchunk, c = e % nchunk;
      *reinterpret_cast<int4*>(Bs + c * N * 16 + n * 16) =
          *reinterpret_cast<const int4*>(B + (size_t)n * kbytes + c * 16);
    }
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr_s;
  if (which == 3 && tid == 0) {
    mbar_expect_tx(&bar[1], N * 32);
    tma_load_3d(Bs, &mapB, &bar[1], 0, 0, 0);
  }
  if (which == 3) mbar_wait(&bar[1], 0);
  if (which == 1) {  // A -> TMEM columns [256, 256 + K/2), 2 bf16 per column
    const uint32_t* row = reinterpret_cast<const uint32_t*>(A + (size_t)tid * kbytes);
    for (int c = 0; c < K / 2; c += 8) {
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = row[c + i];
      tmem_st8(t + ((uint32_t)(warp * 32) << 16) + 256 + c, v);
    }
    tmem_st_wait();
    fence_before();
    __syncthreads();
    fence_after();
  }
  if (tid == 0) {
    if (!i8) {
      const uint32_t id = idesc_bf16(128, N, 0, which == 2 || which == 5);
      for (int j = 0; j < K / 16; ++j) {
        uint64_t bd = which == 2   ? sdesc(smem_u32(Bs) + 2 * j * (N / 8) * 128, (N / 8) * 128, 128)
                      : which == 5 ? sdesc(smem_u32(Bs) + 2 * j * 128, 128, K * 16)
                                   : sdesc(smem_u32(Bs) + 2 * j * N * 16, N * 16, 128);
        if (which == 1) {
          mma_bf16_ts(t, t + 256 + j * 8, bd, id, j > 0);
        } else {
          uint64_t ad = sdesc(smem_u32(As) + 2 * j * 128 * 16, 128 * 16, 128);
          mma_bf16_ss(t, ad, bd, id, j > 0);
        }
      }
    } else {
      const uint32_t id = idesc_i8(128, N);
      mma_i8_ss(t, sdesc(smem_u32(As), 128 * 16, 128), sdesc(smem_u32(Bs), N * 16, 128), id, 0);
    }
    commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  fence_after();
  uint32_t* out = reinterpret_cast<uint32_t*>(D) + (size_t)tid * N;
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(t + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) out[c + i] = r[i];
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(t);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// [rows x 32 bytes] int8 rows -> 3-D map {16 B, rows, 2 chunks}: a box lands
// in shared memory as two chunk slabs [2][box_rows][16 B] (K-major, no swizzle).
bool make_rows32_map(CUtensorMap* map, const void* base, int64_t rows, int box_rows) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {16, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {32, 16};  // bytes, for dims 1 and 2
  cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace tav2

extern "C" int tav2_tc_selftest(int which, const void* A, const void* B, void* D, int N, int K,
                                void* stream) {
  using namespace tav2;
  if (which < 0 || which > 5 || N < 16 || N > 256 || N % 16 || K < 16 || K > 256 || K % 16)
    return TAV2_EINVAL;
  if ((which == 3 || which == 4) && K != 32) return TAV2_EINVAL;
  CUtensorMap map{};
  if (which == 3 && !make_rows32_map(&map, B, N, N)) return TAV2_ECUDA;
  const int esz = (which == 3 || which == 4) ? 1 : 2;
  size_t smem = (size_t)(128 + N) * K * esz + 1024;
  if (cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return TAV2_ECUDA;
  tc_selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(which, (const uint8_t*)A, (const uint8_t*)B,
                                                             D, N, K, map);
  if (cudaGetLastError() != cudaSuccess) return TAV2_ECUDA;
  return cudaStreamSynchronize((cudaStream_t)stream) == cudaSuccess ? TAV2_OK : TAV2_ECUDA;
}
