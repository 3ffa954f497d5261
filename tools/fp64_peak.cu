// fp64_peak.cu -- measure the B200 FP64 pipe peak (DFMA and DADD/DMUL issue
// rates) with independent dependency chains; used as the "alu" roofline
// denominator.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chains(double* out, int iters, double a, double b)
{
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) {  // DFMA
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            } else {        // DADD
                x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
                x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main()
{
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 256, blocks = sms * 8, iters = 2048;
    double* out;
    cudaMalloc(&out, sizeof(double) * threads * blocks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int op = 0; op < 2; ++op) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) chains<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            else chains<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        double inst = (double)threads * blocks * iters * 64;  // thread-level fp64 instructions
        double tinst = inst / (best * 1e-3) / 1e12;
        printf("{\"op\": \"%s\", \"ms\": %.4f, \"thread_inst_per_s_T\": %.3f, \"tflops\": %.3f, \"sms\": %d}\n",
               op == 0 ? "DFMA" : "DADD", best, tinst, op == 0 ? 2 * tinst : tinst, sms);
    }
    return 0;
}
