// mbarrier.test_wait.parity semantics on sm_100a (development check for the producer-in-pencil pump)
#include <cstdio>
__device__ unsigned addr_of(void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ bool test(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok;
}
__device__ bool trywait(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok;
}
__global__ void k(int* out) {
    __shared__ unsigned long long b;
    const unsigned bar = addr_of(&b);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    out[0] = test(bar, 1);  out[1] = test(bar, 0);
    out[2] = trywait(bar, 1); out[3] = trywait(bar, 0);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    out[4] = test(bar, 0); out[5] = test(bar, 1);
}
int main() {
    int* d; cudaMalloc(&d, 64); k<<<1, 1>>>(d); int h[6]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("fresh: test(1)=%d test(0)=%d try(1)=%d try(0)=%d | after arrive: test(0)=%d test(1)=%d | %s\n", h[0], h[1], h[2], h[3], h[4], h[5], cudaGetErrorString(cudaGetLastError()));
}
