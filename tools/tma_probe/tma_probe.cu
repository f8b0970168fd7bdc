// Minimal TMA probe: loads one 2-D box of a u32 plane into shared memory and writes it back.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, int bw, int bh, int cx, int cy, uint32_t* out, int mode) {
    extern __shared__ __align__(128) unsigned char raw[];
    unsigned char* sm = raw + ((128u - (smem_u32(raw) & 127u)) & 127u);
    uint64_t* bar = (uint64_t*)(sm + ((bw * bh * 4 + 127) & ~127));
    uint32_t* buf = (uint32_t*)sm;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bw * bh * 4) : "memory");
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(smem_u32(buf)), "l"(&tmap), "r"(smem_u32(bar)), "r"(cx), "r"(cy) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(smem_u32(buf)), "l"(&tmap), "r"(smem_u32(bar)), "r"(cx), "r"(cy) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(0) : "memory");
    for (int k = threadIdx.x; k < bw * bh; k += blockDim.x) out[k] = buf[k];
}

#include <stdlib.h>
int main(int argc, char** argv) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
    PFN_encodeTiled enc = (PFN_encodeTiled)p;
    printf("encode fn %p q=%d\n", p, (int)q);
    struct Case { int W, H, bw, bh, cx, cy, mode; } cases[] = {
        {256, 64, 68, 26, 2, 0, 0}, {256, 64, 68, 26, 0, -5, 0}, {256, 64, 68, 26, 4, 0, 0}, {256, 64, 68, 26, 1, 3, 0}, {28, 7, 68, 26, 0, 0, 0}, {256, 64, 68, 26, -4, 0, 0},
        {256, 64, 68, 26, 0, 0, 1}, {256, 64, 252, 74, 0, 0, 0}};
    int only = argc > 1 ? atoi(argv[1]) : -1; int ci = -1;
    for (auto c : cases) {
        if (only >= 0 && ++ci != only) continue;
        uint32_t* d = nullptr;
        cudaMalloc(&d, (size_t)c.W * c.H * 4);
        std::vector<uint32_t> h((size_t)c.W * c.H);
        for (size_t i = 0; i < h.size(); ++i) h[i] = (uint32_t)i;
        cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        CUtensorMap m;
        cuuint64_t dims[2] = {(cuuint64_t)c.W, (cuuint64_t)c.H};
        cuuint64_t str[1] = {(cuuint64_t)c.W * 4};
        cuuint32_t box[2] = {(cuuint32_t)c.bw, (cuuint32_t)c.bh};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        uint32_t* o = nullptr;
        cudaMalloc(&o, (size_t)c.bw * c.bh * 4);
        size_t sm = ((c.bw * c.bh * 4 + 127) & ~127) + 256;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        probe<<<1, 128, sm>>>(m, c.bw, c.bh, c.cx, c.cy, o, c.mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint32_t> ho((size_t)c.bw * c.bh);
        int bad = -1;
        if (e == cudaSuccess) {
            cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
            bad = 0;
            for (int yy = 0; yy < c.bh; ++yy)
                for (int xx = 0; xx < c.bw; ++xx) {
                    int gx = c.cx + xx, gy = c.cy + yy;
                    uint32_t want = (gx >= 0 && gx < c.W && gy >= 0 && gy < c.H) ? (uint32_t)(gy * c.W + gx) : 0u;
                    bad += ho[yy * c.bw + xx] != want;
                }
        }
        printf("W=%d H=%d box=%dx%d at (%d,%d) mode=%d encode=%d launch=%s mismatches=%d\n", c.W, c.H, c.bw, c.bh, c.cx,
               c.cy, c.mode, (int)r, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
        cudaFree(d);
        cudaFree(o);
    }
    return 0;
}
