#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(192) plain(int *p) { extern __shared__ uint8_t s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
__global__ void __launch_bounds__(192) withtmem(int *p) {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(128));
    if (p) p[threadIdx.x] = slot;
}
__global__ void __launch_bounds__(192) withpdl(int *p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p) p[threadIdx.x] = 1;
}
int main() {
    int n;
    for (size_t d : {0, 60000, 99440}) {
        cudaFuncSetAttribute(plain, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        cudaFuncSetAttribute(withtmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, plain, 192, d); printf("plain dyn %zu: %d\n", d, n);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, withtmem, 192, d); printf("tmem dyn %zu: %d\n", d, n);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, withpdl, 192, d); printf("pdl dyn %zu: %d\n", d, n);
    }
}
