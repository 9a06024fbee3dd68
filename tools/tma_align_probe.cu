// tma_align_probe.cu -- does a 2-D SWIZZLE_128B TMA load whose shared-memory destination is only
// 128-byte aligned (k*128 bytes past a 1024-byte boundary) write the absolute-address swizzle
// pattern (16-byte chunk c of the row at address X lands at chunk c ^ ((X >> 7) & 7))?  The
// stacked-halo tiles of the 13x13 layers place one image row (14 pixels = 1792 bytes) per box.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma_align_probe tools/tma_align_probe.cu && /tmp/tma_align_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

typedef CUresult (*PFN_tiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int R = 14;   // box rows (one 13x13 image row + pad = 14 pixels of 64 channels)

__global__ void probe(const __grid_constant__ CUtensorMap map, uint16_t* out, int k, int row0) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    uint4* z = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < 4096 / 16; i++) z[i] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(R * 128) : "memory");
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + 128 * k);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(b), "r"(0), "r"(row0)
            : "memory");
        asm volatile(
            "{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(b)
            : "memory");
    }
    __syncthreads();
    const uint16_t* s16 = reinterpret_cast<const uint16_t*>(smem);
    for (int i = threadIdx.x; i < 4096 / 2; i += blockDim.x) out[i] = s16[i];
}

int main() {
    PFN_tiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no encoder\n"); return 1; }
    const int rows = 64;
    std::vector<uint16_t> h(rows * 64);
    for (int r = 0; r < rows; r++)
        for (int c = 0; c < 64; c++) h[r * 64 + c] = (uint16_t)(r * 64 + c + 1);   // nonzero tags
    uint16_t *dA, *dO;
    cudaMalloc(&dA, h.size() * 2);
    cudaMalloc(&dO, 4096);
    cudaMemcpy(dA, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[2] = {64, (cuuint64_t)rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, R};
    cuuint32_t es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
    }
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    int bad_total = 0;
    for (int k = 0; k < 8; k++) {
        const int row0 = 3 + k;
        probe<<<1, 128, 8192>>>(map, dO, k, row0);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("k=%d: %s\n", k, cudaGetErrorString(e)); return 2; }
        std::vector<uint16_t> o(2048);
        cudaMemcpy(o.data(), dO, 4096, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < R; r++) {
            const int X = (k + r) * 128;                 // row address relative to the 1024-aligned base
            for (int c = 0; c < 64; c++) {
                const int chunk = (c / 8) ^ ((X >> 7) & 7);
                const int pos = (X + chunk * 16) / 2 + (c % 8);
                if (o[pos] != h[(row0 + r) * 64 + c]) bad++;
            }
        }
        printf("k=%d (dst %d B past a 1024-byte boundary): %s (%d mismatches)\n", k, 128 * k,
               bad ? "NOT absolute swizzle" : "absolute-address swizzle", bad);
        bad_total += bad;
    }
    printf(bad_total ? "RESULT: misaligned TMA destinations do not follow the absolute pattern\n"
                     : "RESULT: 128-byte-aligned TMA destinations follow the absolute-address swizzle\n");
    return 0;
}
