// Staging from the HBM-resident feature store (tav2_store_*):
// one launch copies every stored user's token run (emb i8[32], action u16,
// surface u8 per token) from the store pool into the staged token columns,
// instead of three cudaMemcpyAsync per user.  HBM-bound: 70 B of traffic per
// token (35 B read + 35 B written); 16-byte vectors for the embeddings.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"

namespace tav2 {

constexpr int kGatherThreads = 256;

// grid (x: token chunks of one run, y: run); a token's 32-byte embedding row is
// two int4, so each thread moves 16 B of embeddings per step
__global__ void __launch_bounds__(kGatherThreads)
    store_gather_kernel(const StoreCopy* __restrict__ d, const int8_t* __restrict__ semb,
                        const uint16_t* __restrict__ sact, const uint8_t* __restrict__ ssurf,
                        int8_t* __restrict__ demb, uint16_t* __restrict__ dact, uint8_t* __restrict__ dsurf) {
  const StoreCopy c = d[blockIdx.y];
  const int stride = gridDim.x * kGatherThreads;
  const int t0 = blockIdx.x * kGatherThreads + threadIdx.x;
  const int4* se = reinterpret_cast<const int4*>(semb + c.src * kEmbed);
  int4* de = reinterpret_cast<int4*>(demb + c.dst * kEmbed);
  for (int i = t0; i < 2 * c.n; i += stride) de[i] = __ldg(se + i);
  for (int i = t0; i < c.n; i += stride) {
    dact[c.dst + i] = __ldg(sact + c.src + i);
    dsurf[c.dst + i] = __ldg(ssurf + c.src + i);
  }
}

cudaError_t launch_store_gather(const StoreCopy* d, int n, int max_tok, const int8_t* semb,
                                const uint16_t* sact, const uint8_t* ssurf, int8_t* demb, uint16_t* dact,
                                uint8_t* dsurf, cudaStream_t s) {
  if (n == 0 || max_tok == 0) return cudaSuccess;
  const dim3 grid((2 * max_tok + kGatherThreads - 1) / kGatherThreads, n);
  store_gather_kernel<<<grid, kGatherThreads, 0, s>>>(d, semb, sact, ssurf, demb, dact, dsurf);
  return cudaGetLastError();
}

}  // namespace tav2
