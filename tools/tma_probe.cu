// Standalone probe: 3-D TMA box load into shared memory (debug tool).
// usage: tma_probe <variant>   0: param desc, shared::cluster  1: param desc, shared::cta
//                               2: global-memory desc            3: small box 32x8x8
//                               4: param desc + fence.proxy.async instead of mbarrier_init fence
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tmap, const CUtensorMap *gmap, float *out, int nbox, int variant, int cx, int cy, int cz, int shift) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float *box = (float *)sm;
    uint64_t *bar = (uint64_t *)(sm + nbox * 4 + 4096);
    const CUtensorMap *m = variant == 2 ? gmap : &tmap;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(bar)), "r"(1));
        if (variant == 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        else asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(nbox * 4) : "memory");
        if (variant == 1)
            asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(box)), "l"((uint64_t)m), "r"(cx), "r"(cx), "r"(cx), "r"(su(bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(box + shift)), "l"((uint64_t)m), "r"(cx), "r"(cy), "r"(cz), "r"(su(bar)) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su(bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < nbox; i += blockDim.x) out[i] = box[i];
}
typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                        const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char **argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    int BX = getenv("BXW") ? atoi(getenv("BXW")) : 36, BY = 18, BZ = 18;
    if (variant == 3) { BX = 32; BY = 8; BZ = 8; }
    int nbox = BX * BY * BZ;
    int d[3] = {64, 64, 64};
    void *fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, nbox * 4 + 8192);
    size_t n = (size_t)d[0] * d[1] * d[2];
    std::vector<float> h(n); for (size_t i = 0; i < n; ++i) h[i] = (float)i;
    float *g, *o; cudaMalloc(&g, n * 4); cudaMalloc(&o, nbox * 4);
    cudaMemcpy(g, h.data(), n * 4, cudaMemcpyHostToDevice);
    CUtensorMap m; memset(&m, 0, sizeof(m));
    cuuint64_t gd[3] = {(cuuint64_t)d[0], (cuuint64_t)d[1], (cuuint64_t)d[2]};
    cuuint64_t gs[2] = {(cuuint64_t)d[0] * 4, (cuuint64_t)d[0] * d[1] * 4};
    cuuint32_t bd[3] = {(cuuint32_t)BX, (cuuint32_t)BY, (cuuint32_t)BZ}, es[3] = {1, 1, 1};
    CUresult r = ((Enc)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, getenv("NANFILL") ? CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA : CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap *gm; cudaMalloc(&gm, sizeof(m)); cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    int cx = argc > 2 ? atoi(argv[2]) : -1;
    int cy = argc > 4 ? atoi(argv[4]) : cx, cz = argc > 5 ? atoi(argv[5]) : cx;
    if (variant == 5) { CUresult r2 = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); printf("direct enc %d\n", (int)r2); }
    printf("q=%d desc:", (int)q); for (int i = 0; i < 16; ++i) printf(" %016llx", (unsigned long long)((unsigned long long*)&m)[i]); printf("\n");
    int shift = argc > 3 ? atoi(argv[3]) : 0;
    k<<<1, 256, nbox * 4 + 8192>>>(m, gm, o, nbox, variant, cx, cy, cz, shift);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(nbox); cudaMemcpy(ho.data(), o, nbox * 4, cudaMemcpyDeviceToHost);
    printf("shift %d: ", shift);
    printf("variant %d box %dx%dx%d enc %d run %s  box[1,1,1]=%g (expect 0) box[2,1,1]=%g (expect 1) box[0]=%g\n", variant,
           BX, BY, BZ, (int)r, cudaGetErrorString(e), ho[(1 * BY + 1) * BX + 1 + shift], ho[(1 * BY + 1) * BX + 2 + shift], ho[shift]);
    // first mismatch against the expected field value (NaN / 0 outside the domain)
    int bad = 0;
    for (int z = 0; z < BZ && !bad; ++z) for (int y = 0; y < BY && !bad; ++y) for (int x = 0; x < BX; ++x) {
        int gx = cx + x, gy = cy + y, gz = cz + z;
        bool in = gx >= 0 && gx < d[0] && gy >= 0 && gy < d[1] && gz >= 0 && gz < d[2];
        float v = ho[(z * BY + y) * BX + x + shift];
        float want = in ? (float)((size_t)(gz * d[1] + gy) * d[0] + gx) : 0.f;
        bool ok = in ? v == want : (getenv("NANFILL") ? v != v : v == 0.f);
        if (!ok) { printf("mismatch at box (%d,%d,%d): %g want %s%g\n", x, y, z, v, in ? "" : "oob ", want); bad = 1; break; }
    }
    printf("coords (%d,%d,%d) bx %d: %s\n", cx, cy, cz, BX, bad ? "BAD" : "all cells ok");
    return e != cudaSuccess;
}
