// tma_probe.cu -- minimal TMA 4-D load probe (debugging aid, not part of the library).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void probe(const __grid_constant__ CUtensorMap tm, double *out, int x0, int y0, int z, int bytes = 34 * 10 * 6 * 8) {
    extern __shared__ __align__(128) unsigned char raw[];
    double *buf = (double *)raw;
    uint64_t *bar = (uint64_t *)(raw + 34 * 10 * 6 * 8 + 64);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        if (VARIANT == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else if (VARIANT == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(z), "r"(0), "r"(smem_u32(bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(0) : "memory");
    }
    for (int q = threadIdx.x; q < 34 * 10 * 6; q += blockDim.x) out[q] = buf[q];
}

int main(int argc, char **argv) {
    const int V = argc > 1 ? atoi(argv[1]) : 0;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    const int nx = 37, ny = 23, nz = 11, px = 64;
    size_t cs = (size_t)px * ny * nz;
    std::vector<double> h(6 * cs);
    for (size_t q = 0; q < h.size(); ++q) h[q] = (double)q;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 34 * 10 * 6 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz, 6};
    cuuint64_t str[3] = {(cuuint64_t)px * 8, (cuuint64_t)px * ny * 8, cs * 8};
    cuuint32_t box[4] = {(cuuint32_t)(V == 4 ? 32 : 34), 10, 1, (cuuint32_t)(V == 5 ? 1 : 6)}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode=%d qr=%d\n", (int)r, (int)qr);
    int smem = 34 * 10 * 6 * 8 + 128;
    for (int v = V; v <= V; ++v) {
        const int c0 = V == 3 ? 0 : -1;
        const int cx = argc > 2 ? atoi(argv[2]) : c0, cy = argc > 3 ? atoi(argv[3]) : c0, cz = argc > 4 ? atoi(argv[4]) : 2;
        const int bytes = (int)(box[0] * box[1] * box[3] * 8);
        if (v == 1) probe<1><<<1, 128, smem>>>(tm, o, cx, cy, cz, bytes);
        else if (v == 2) probe<2><<<1, 128, smem>>>(tm, o, cx, cy, cz, bytes);
        else probe<0><<<1, 128, smem>>>(tm, o, cx, cy, cz, bytes);
        cudaError_t e = cudaDeviceSynchronize();
        printf("variant %d: %s\n", v, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<double> ho(34 * 10 * 6);
        cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
        // element (x=0 -> global -1 => 0), (x=1,y=1) -> global (0,0,2,comp0)
        printf("  box[0]=%g box[1*34+1]=%g expect %g ; comp1 %g expect %g\n", ho[0], ho[34 + 1],
               (double)(0 + px * (0 + ny * 2)), ho[340 + 34 + 1], (double)(cs + px * ny * 2));
    }
    return 0;
}
