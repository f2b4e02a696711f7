// Staging from the HBM-resident feature store (tav2_store_*):
// one launch copies every stored user's token run (emb i8[32], action u16,
// surface u8 per token) from the store pool into the staged token columns,
// instead of three cudaMemcpyAsync per user.  HBM-bound: 70 B of traffic per
// token (35 B read + 35 B written); 32-byte vectors for the embeddings.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tav2_common.cuh"

namespace tav2 {

constexpr int kGatherThreads = 256;

// grid (x: token chunks of one run, y: run); thread = token: its 32-byte
// embedding row moves as one 256-bit load / store (LDG.256 / STG.256), then
// its action and surface
__global__ void __launch_bounds__(kGatherThreads)
    store_gather_kernel(const StoreCopy* __restrict__ d, const int8_t* __restrict__ semb,
                        const uint16_t* __restrict__ sact, const uint8_t* __restrict__ ssurf,
                        int8_t* __restrict__ demb, uint16_t* __restrict__ dact, uint8_t* __restrict__ dsurf) {
  const StoreCopy c = d[blockIdx.y];
  const int stride = gridDim.x * kGatherThreads;
  for (int i = blockIdx.x * kGatherThreads + threadIdx.x; i < c.n; i += stride) {
    uint32_t r[8];
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(semb + (c.src + i) * kEmbed));
    const uint16_t a = __ldg(sact + c.src + i);
    const uint8_t sf = __ldg(ssurf + c.src + i);
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(demb + (c.dst + i) * kEmbed), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
    dact[c.dst + i] = a;
    dsurf[c.dst + i] = sf;
  }
}

cudaError_t launch_store_gather(const StoreCopy* d, int n, int max_tok, const int8_t* semb,
                                const uint16_t* sact, const uint8_t* ssurf, int8_t* demb, uint16_t* dact,
                                uint8_t* dsurf, cudaStream_t s) {
  if (n == 0 || max_tok == 0) return cudaSuccess;
  const dim3 grid((max_tok + kGatherThreads - 1) / kGatherThreads, n);
  store_gather_kernel<<<grid, kGatherThreads, 0, s>>>(d, semb, sact, ssurf, demb, dact, dsurf);
  return cudaGetLastError();
}

}  // namespace tav2
