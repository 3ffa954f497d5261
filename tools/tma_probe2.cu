// TMA through libcu++ (cuda::barrier + cp_async_bulk_tensor_3d_global_to_shared), the
// CUDA Programming Guide's pattern, as a reference for tools/tma_probe.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda/barrier>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
using barrier = cuda::barrier<cuda::thread_scope_block>;
namespace cde = cuda::device::experimental;

__global__ void k(const __grid_constant__ CUtensorMap m, double* out, int x0, int y0, int z0, int bx)
{
    __shared__ alignas(128) double buf[34 * 10];
#pragma nv_diag_suppress static_var_with_dynamic_init
    __shared__ barrier bar;
    if (threadIdx.x == 0) {
        init(&bar, blockDim.x);
        cde::fence_proxy_async_shared_cta();
    }
    __syncthreads();
    barrier::arrival_token token;
    if (threadIdx.x == 0) {
        if (z0 >= 0) cde::cp_async_bulk_tensor_3d_global_to_shared(buf, &m, x0, y0, z0, bar);
        else cde::cp_async_bulk_tensor_2d_global_to_shared(buf, &m, x0, y0, bar);
        token = cuda::device::barrier_arrive_tx(bar, 1, bx * 10 * 8);
    } else {
        token = bar.arrive();
    }
    bar.wait(std::move(token));
    for (int q = threadIdx.x; q < 340; q += blockDim.x) out[q] = buf[q];
}

int main(int argc, char** argv)
{
    const int dtk = argc > 1 ? atoi(argv[1]) : 0, bx = argc > 2 ? atoi(argv[2]) : 34, rank = argc > 3 ? atoi(argv[3]) : 3;
    const int nx = 40, ny = 12, nz = 5;
    std::vector<double> h(nx * ny * nz);
    for (size_t q = 0; q < h.size(); ++q) h[q] = 1.0 + q;
    double *dg, *dout;
    cudaMalloc(&dg, h.size() * 8);
    cudaMalloc(&dout, 340 * 8);
    cudaMemcpy(dg, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    if (argc > 4) enc = cuTensorMapEncodeTiled;  // linked from libcuda
    int dv = 0, rv = 0;
    cudaDriverGetVersion(&dv);
    cudaRuntimeGetVersion(&rv);
    printf("driver %d runtime %d entry %p direct %p\n", dv, rv, fn, (void*)cuTensorMapEncodeTiled);
    CUtensorMap m;
    const cuuint64_t dims[3] = {nx, ny, nz}, str[2] = {nx * 8, nx * ny * 8};
    const cuuint32_t box[3] = {(cuuint32_t)bx, 10, 1}, es[3] = {1, 1, 1};
    const CUtensorMapDataType dts[3] = {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_DATA_TYPE_INT64, CU_TENSOR_MAP_DATA_TYPE_UINT64};
    CUresult r = enc(&m, dts[dtk], rank, dg, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    k<<<1, 128>>>(m, dout, 3, 1, rank == 3 ? 2 : -1, bx);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> o(340);
    cudaMemcpy(o.data(), dout, 340 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < 10; ++y)
        for (int x = 0; x < 34; ++x) {
            const int gx = 3 + x, gy = 1 + y;
            const double want = (gx < nx && gy < ny) ? h[gx + nx * (gy + ny * 2)] : 0.0;
            bad += o[y * 34 + x] != want;
        }
    printf("libcu++ TMA dtype %d box %d rank %d: %s, mismatches %d\n", dtk, bx, rank, cudaGetErrorString(e), bad);
    return bad != 0;
}
