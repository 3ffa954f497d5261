// fp64_latency.cu -- FP64 dependent-chain latency and throughput vs. warps / ILP on one SM
// (explains the latency-bound behaviour of the SALE kernels).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, int iters, double a, double b, long long* cyc)
{
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-3 + k;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
    }
    long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
void run(int warps, double* out, long long* dcyc)
{
    const int iters = 4096;
    chain<ILP><<<1, 32 * warps>>>(out, iters, 0.999999, 1e-7, dcyc);
    long long cyc;
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    double per_instr = (double)cyc / (iters * 2.0 * ILP);         // cycles per dependent-chain instr (one warp)
    double sm_rate = 2.0 * ILP * iters * warps / (double)cyc;     // warp fp64 instr per cycle per SM
    printf("{\"ilp\": %d, \"warps\": %d, \"cycles_per_instr_per_warp\": %.2f, \"sm_warp_fp64_per_cycle\": %.3f}\n",
           ILP, warps, per_instr, sm_rate);
}

int main()
{
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8 * 1024 * 32);
    cudaMalloc(&cyc, 8);
    int ws[] = {1, 4, 8, 16, 32};
    for (int w : ws) run<1>(w, out, cyc);
    for (int w : ws) run<2>(w, out, cyc);
    for (int w : ws) run<4>(w, out, cyc);
    return 0;
}
