// Standalone check of the TMA path kr_tail_tma uses: a cuTensorMapEncodeTiled 3-D fp64
// map, cp.async.bulk.tensor.3d into shared memory completing on an mbarrier, out-of-range
// zero fill.  nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

struct Maps { CUtensorMap a; };

__global__ void k(const __grid_constant__ Maps m, const CUtensorMap* gmap, double* out, int x0, int y0, int z0)
{
    const CUtensorMap* map = gmap ? gmap : &m.a;
    __shared__ alignas(128) double buf[34 * 10];
    __shared__ alignas(8) unsigned long long bar;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned d = (unsigned)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(34 * 10 * 8) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d),
            "l"(reinterpret_cast<unsigned long long>(map)), "r"(x0), "r"(y0), "r"(z0), "r"(b)
            : "memory");
    }
    unsigned done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(b), "r"(0u) : "memory");
    } while (!done);
    for (int q = threadIdx.x; q < 340; q += blockDim.x) out[q] = buf[q];
}

int main()
{
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
    Maps m;
    const cuuint64_t dims[3] = {nx, ny, nz}, str[2] = {nx * 8, nx * ny * 8};
    const cuuint32_t box[3] = {34, 10, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dg, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    int bad = 0;
    CUtensorMap* gm = nullptr;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m.a, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    const int cases[3][3] = {{3, 1, 2}, {-2, -2, 0}, {10, 5, 4}};
    for (int mode = 1; mode >= 0; --mode)
    for (auto& c : cases) {
        k<<<1, 128>>>(m, mode ? gm : nullptr, dout, c[0], c[1], c[2]);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> o(340);
        cudaMemcpy(o.data(), dout, 340 * 8, cudaMemcpyDeviceToHost);
        for (int y = 0; y < 10; ++y)
            for (int x = 0; x < 34; ++x) {
                const int gx = c[0] + x, gy = c[1] + y, gz = c[2];
                const double want = (gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? h[gx + nx * (gy + ny * gz)] : 0.0;
                bad += o[y * 34 + x] != want;
            }
        printf("mode %s case (%d,%d,%d): %s, mismatches so far %d\n", mode ? "global map" : "param map", c[0], c[1], c[2], cudaGetErrorString(e), bad);
    }
    return bad != 0;
}
