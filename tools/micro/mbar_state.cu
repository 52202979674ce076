#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ unsigned long long rd(unsigned long long* b) { unsigned long long v; asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(b)) : "memory"); return v; }
__device__ bool tryw(unsigned long long* b, uint32_t ph) { uint32_t ok; asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory"); return ok; }
__global__ void k() {
  __shared__ unsigned long long bar[4];
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  printf("init       %016llx try0=%d\n", rd(&bar[0]), tryw(&bar[0], 0));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(0) : "memory");
  printf("arrive tx0 %016llx try0=%d try1=%d\n", rd(&bar[0]), tryw(&bar[0], 0), tryw(&bar[0], 1));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(336) : "memory");
  printf("arrive tx336 %016llx try0=%d try1=%d\n", rd(&bar[0]), tryw(&bar[0], 0), tryw(&bar[0], 1));
}
int main() { k<<<1, 1>>>(); printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize())); }
