// micro: the big-row pull's per-warp 3-copy TMA item staging, isolated
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ bool mbar_try(unsigned long long* b, uint32_t phase) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(phase) : "memory");
  return ok != 0;
}
struct alignas(16) ItemStage {
  unsigned long long bar[2];
  uint32_t other[2][136];
  uint32_t mask[2][136];
  uint8_t batch[2][160];
  unsigned long long beg[2], end[2];
  uint32_t u[2], own[2];
};
__global__ void k(const uint32_t* other, const uint32_t* mask, const uint8_t* batch, const unsigned long long* begs, int nch, unsigned long long* sum, int variant) {
  __shared__ unsigned long long pad[1900];
  extern __shared__ __align__(128) unsigned long long dyn[];
  ItemStage* stg = reinterpret_cast<ItemStage*>(dyn + 8 * 520) + (threadIdx.x >> 5);
  const unsigned lane = threadIdx.x & 31;
  const unsigned nw = gridDim.x * blockDim.x / 32, my = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (lane == 0) pad[threadIdx.x / 32] = 0;
  if (my >= nch) return;
  if (lane == 0) { mbar_init(&stg->bar[0]); mbar_init(&stg->bar[1]); fence_mbar_init(); }
  __syncwarp();
  auto issue = [&](int si, unsigned long long b, unsigned long long e) {
    stg->beg[si] = b; stg->end[si] = e;
    const unsigned long long a4 = b & ~3ull, e4 = (e + 3) & ~3ull, a16 = b & ~15ull, e16 = (e + 15) & ~15ull;
    const uint32_t b4 = uint32_t(e4 - a4) * 4, b1 = uint32_t(e16 - a16);
    mbar_expect_tx(&stg->bar[si], 2 * b4 + b1);
    bulk_g2s(stg->other[si], other + a4, b4, &stg->bar[si]);
    bulk_g2s(stg->mask[si], mask + a4, b4, &stg->bar[si]);
    if (variant == 0) bulk_g2s(stg->batch[si], batch + a16, b1, &stg->bar[si]);
    else bulk_g2s(stg->batch[si], batch + a16, b1, &stg->bar[si]);
  };
  if (lane == 0) issue(0, begs[my], begs[my + 1]);
  unsigned long long acc = 0; uint32_t it = 0;
  for (unsigned c = my; c < nch; c += nw, ++it) {
    __syncwarp();
    int si = it & 1;
    if (lane == 0 && c + nw < nch) issue(si ^ 1, begs[c + nw], begs[c + nw + 1]);
    long spins = 0;
    while (!mbar_try(&stg->bar[si], (it >> 1) & 1)) if (++spins == 1000000) { if (lane == 0) printf("stuck warp %u it %u beg %llu end %llu\n", my, it, stg->beg[si], stg->end[si]); __trap(); }
    const unsigned long long b = stg->beg[si], e = stg->end[si];
    const uint32_t o4 = b & 3, o16 = b & 15;
    for (uint32_t i = lane; i < e - b; i += 32) acc += stg->other[si][o4 + i] + stg->mask[si][o4 + i] + stg->batch[si][o16 + i];
  }
  atomicAdd(sum, acc);
}
int main() {
  const int M = 1 << 20, nch = 8000;
  uint32_t *o, *m; uint8_t* b; unsigned long long *begs, *sum;
  cudaMalloc(&o, M * 4 + 256); cudaMalloc(&m, M * 4 + 256); cudaMalloc(&b, M + 256); cudaMalloc(&begs, (nch + 1) * 8); cudaMalloc(&sum, 8);
  uint32_t* h = new uint32_t[M]; uint8_t* hb = new uint8_t[M]; unsigned long long* hbeg = new unsigned long long[nch + 1];
  for (int i = 0; i < M; ++i) { h[i] = i; hb[i] = i & 255; }
  unsigned long long x = 0; for (int c = 0; c <= nch; ++c) { hbeg[c] = x; x += 33 + (c * 7919) % 96; }
  cudaMemcpy(o, h, M * 4, cudaMemcpyHostToDevice); cudaMemcpy(m, h, M * 4, cudaMemcpyHostToDevice); cudaMemcpy(b, hb, M, cudaMemcpyHostToDevice);
  cudaMemcpy(begs, hbeg, (nch + 1) * 8, cudaMemcpyHostToDevice); cudaMemset(sum, 0, 8);
  const size_t smem = 8 * 520 * 8 + 8 * sizeof(ItemStage);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148 * 3, 256, smem>>>(o, m, b, begs, nch, sum, 0);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  unsigned long long s = 0, want = 0; cudaMemcpy(&s, sum, 8, cudaMemcpyDeviceToHost);
  for (int c = 0; c < nch; ++c) for (unsigned long long i = hbeg[c]; i < hbeg[c + 1]; ++i) want += 2ull * h[i] + hb[i];
  printf("sum %llu want %llu\n", s, want);
}
