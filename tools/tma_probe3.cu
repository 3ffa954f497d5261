// Non-tensor bulk copy (cp.async.bulk global -> shared, mbarrier complete_tx), and a
// plain mbarrier arrive/wait, to isolate what tools/tma_probe*.cu trip over.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__global__ void k(const double* src, double* out, int mode)
{
    __shared__ alignas(128) double buf[256];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned d = (unsigned)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
        if (mode >= 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode >= 2) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2048) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                         "l"(src), "r"(2048), "r"(b)
                         : "memory");
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
        }
    }
    unsigned done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(b), "r"(0u) : "memory");
    } while (!done);
    if (mode >= 2) out[threadIdx.x] = buf[threadIdx.x];
}

int main(int argc, char** argv)
{
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    double *src, *out;
    cudaMalloc(&src, 2048);
    cudaMalloc(&out, 2048);
    double h[256];
    for (int q = 0; q < 256; ++q) h[q] = q + 0.5;
    cudaMemcpy(src, h, 2048, cudaMemcpyHostToDevice);
    k<<<1, 256>>>(src, out, mode);
    cudaError_t e = cudaDeviceSynchronize();
    double o[256] = {0};
    cudaMemcpy(o, out, 2048, cudaMemcpyDeviceToHost);
    int bad = 0;
    if (mode >= 2)
        for (int q = 0; q < 256; ++q) bad += o[q] != h[q];
    printf("mode %d: %s, mismatches %d\n", mode, cudaGetErrorString(e), bad);
    return 0;
}
