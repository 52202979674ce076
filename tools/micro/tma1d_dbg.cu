// micro test of the 1D TMA + mbarrier helpers used by simulate's big-row pull
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
struct alignas(16) St { unsigned long long bar[2]; uint32_t d[2][136]; };
__global__ void k(const uint32_t* src, uint32_t* out, int n) {
  extern __shared__ unsigned long long dyn[];
  St* s = reinterpret_cast<St*>(dyn + 8);
  const unsigned lane = threadIdx.x & 31;
  if (lane == 0) { mbar_init(&s->bar[0]); mbar_init(&s->bar[1]); fence_mbar_init(); printf("after init %llx\n", s->bar[0]); mbar_expect_tx(&s->bar[1], 336); printf("after expect 336 %llx\n", s->bar[1]); }
  __syncwarp();
  if (lane == 0) { mbar_expect_tx(&s->bar[0], 512); bulk_g2s(s->d[0], src, 512, &s->bar[0]); }
  for (int it = 0; it < n; ++it) {
    __syncwarp();
    int si = it & 1;
    if (lane == 0 && it + 1 < n) { if (it == 0) { printf("bar1 before expect %llx\n", s->bar[1]); } mbar_expect_tx(&s->bar[si ^ 1], 512); bulk_g2s(s->d[si ^ 1], src + (it + 1) * 128, 512, &s->bar[si ^ 1]); }
    long spins = 0;
    while (!mbar_try(&s->bar[si], (it >> 1) & 1)) { if (++spins > 100000000) { if (lane == 0) printf("stuck it=%d\n", it); return; } }
    out[it * 128 + lane] = s->d[si][lane];
    if (lane == 0 && it < 3) printf("it %d done state %llx\n", it, s->bar[si]);
  }
}
int main() {
  uint32_t *src, *out; int n = 10;
  cudaMalloc(&src, n * 512); cudaMalloc(&out, n * 512);
  uint32_t h[1280]; for (int i = 0; i < 1280; ++i) h[i] = i;
  cudaMemcpy(src, h, n * 512, cudaMemcpyHostToDevice); cudaMemset(out, 0, n * 512);
  k<<<1, 32, 4096>>>(src, out, n);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(h, out, n * 512, cudaMemcpyDeviceToHost);
  int bad = 0; for (int it = 0; it < n; ++it) for (int l = 0; l < 32; ++l) bad += h[it * 128 + l] != uint32_t(it * 128 + l);
  printf("bad %d\n", bad);
}
