// desc_probe.cu -- does a tcgen05 SW128 shared-memory descriptor whose start address is shifted by
// r 128-byte rows (not a multiple of the 1024-byte swizzle atom) address the rows r, r+1, ... of a
// tile that was written with the absolute-address 128B swizzle (as TMA writes it)?  Tests K-major
// A shifted along M (halo implicit GEMM: one smem tile reused by every filter tap) and MN-major A
// shifted along K (weight gradient: taps shift the pixel/reduction index), each with the
// descriptor base-offset field 0 and (addr >> 7) & 7.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/desc_probe tools/desc_probe.cu && /tmp/desc_probe
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t base_off) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)(base_off & 7) << 49) | (2ull << 61);
}

constexpr int ROWS = 256;     // smem rows of 128 B (64 bf16) for A
constexpr int N = 16;         // MMA N

// mode 2: A MN-major, one tile of ROWS k-rows x 64 m; M chunk 0 starts at row r, chunk 1 at row r+d
//         (LBO = d*128 bytes, not a multiple of the 1024-byte atom): D[m][n] = sum_k T[r+(m/64)*d+k][m%64]*B[n][k]
// mode 0: A K-major, M rows shifted by r.   D[m][n] = sum_k A[r+m][k] * B[n][k]  (K = 64)
// mode 1: A MN-major, K rows shifted by r.  D[m][n] = sum_k A[r+k][m] * B[n][k]  (M = 64 per chunk x2? use M=128: 2 chunks)
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int mode, int r, int use_base, int d) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sa = smem;                          // mode 0: ROWS x 128 B; mode 1: 2 chunks x ROWS x 128 B
    uint8_t* sb = smem + 2 * ROWS * 128;         // N rows x 128 B (K-major B, K = 64)
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_holder;
    const int tid = threadIdx.x;
    // write A/B with the absolute-address 128B swizzle: 16-byte chunk c of the 128-byte row at
    // address X goes to chunk c ^ ((X >> 7) & 7)
    auto put = [&](uint8_t* rowbase, int c16, const uint4& v) {
        const uint32_t addr = smem_u32(rowbase);
        const int pc = c16 ^ ((addr >> 7) & 7);
        *reinterpret_cast<uint4*>(rowbase + pc * 16) = v;
    };
    const int nchunkA = mode == 1 ? 2 : 1;
    for (int i = tid; i < nchunkA * ROWS * 8; i += blockDim.x) {
        const int ch = i / (ROWS * 8), row = (i / 8) % ROWS, c16 = i % 8;
        uint4 v;
        // mode 0: A row = m (global A is ROWS x 64, K contiguous); mode 1: A row = k, 64 m per chunk
        if (mode == 0 || mode == 2) v = *reinterpret_cast<const uint4*>(A + row * 64 + c16 * 8);
        else v = *reinterpret_cast<const uint4*>(A + row * 128 + ch * 64 + c16 * 8);   // A global: ROWS(k) x 128(m)
        put(sa + ch * ROWS * 128 + row * 128, c16, v);
    }
    for (int i = tid; i < N * 8; i += blockDim.x) {
        const int row = i / 8, c16 = i % 8;
        put(sb + row * 128, c16, *reinterpret_cast<const uint4*>(B + row * 64 + c16 * 8));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_holder;
    if (tid == 0) {
        // idesc: D f32, A/B bf16, a_major (bit 15) = mode, b K-major, N>>3 at 17, M>>4 at 24 (M = 128)
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(mode != 0) << 15) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        for (int k = 0; k < 4; k++) {   // K = 64 in 4 steps of 16
            uint64_t ad;
            if (mode == 0) {
                const uint32_t s = smem_u32(sa) + r * 128 + k * 32;
                ad = desc_sw128(s, 16, 1024, use_base ? ((s >> 7) & 7) : 0);
            } else if (mode == 1) {
                const uint32_t s = smem_u32(sa) + (r + k * 16) * 128;
                ad = desc_sw128(s, ROWS * 128, 1024, use_base ? ((s >> 7) & 7) : 0);
            } else {
                const uint32_t s = smem_u32(sa) + (r + k * 16) * 128;
                ad = desc_sw128(s, d * 128, 1024, 0);
            }
            const uint32_t sbb = smem_u32(sb) + k * 32;
            const uint64_t bd = desc_sw128(sbb, 16, 1024, 0);
            const uint32_t acc = k > 0;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    // wait
    {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(smem_u32(&bar)));
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid < 128) {
        const int w = tid / 32;
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tmem + ((uint32_t)(w * 32) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; j++) D[tid * N + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
    const int AE = ROWS * 128;   // enough for both modes
    std::vector<__nv_bfloat16> hA(AE), hB(N * 64);
    std::vector<float> fA(AE), fB(N * 64);
    srand(1);
    for (int i = 0; i < AE; i++) { float v = (float)(rand() % 17 - 8); hA[i] = __float2bfloat16(v); fA[i] = v; }
    for (int i = 0; i < N * 64; i++) { float v = (float)(rand() % 9 - 4); hB[i] = __float2bfloat16(v); fB[i] = v; }
    __nv_bfloat16 *dA, *dB;
    float* dD;
    cudaMalloc(&dA, AE * 2); cudaMalloc(&dB, N * 64 * 2); cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dA, hA.data(), AE * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), N * 64 * 2, cudaMemcpyHostToDevice);
    const int smem = 2 * ROWS * 128 + N * 128 + 2048;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> hD(128 * N);
    // mode 2: chunk offsets d (rows) of 1, 3, 31, 57 and 8, for shifts r
    for (int d : {1, 3, 8, 31, 57}) {
        int bad = 0;
        for (int r = 0; r < 16; r++) {
            cudaMemset(dD, 0, 128 * N * 4);
            probe<<<1, 128, smem>>>(dA, dB, dD, 2, r, 0, d);
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); return 1; }
            cudaMemcpy(hD.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0;
            for (int m = 0; m < 128; m++)
                for (int n = 0; n < N; n++) {
                    double ref = 0;
                    for (int k = 0; k < 64; k++) ref += (double)fA[(r + (m / 64) * d + k) * 64 + (m % 64)] * fB[n * 64 + k];
                    maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
                }
            if (maxerr > 0) bad++;
        }
        printf("==> mode 2 (MN-major, chunk LBO = %d rows): %d of 16 shifts wrong\n", d, bad);
    }
    for (int mode = 0; mode < 2; mode++)
        for (int use_base = 0; use_base < 2; use_base++) {
            int bad_shifts = 0;
            for (int r = 0; r < 16; r++) {
                cudaMemset(dD, 0, 128 * N * 4);
                probe<<<1, 128, smem>>>(dA, dB, dD, mode, r, use_base, 0);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
                cudaMemcpy(hD.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost);
                double maxerr = 0;
                for (int m = 0; m < 128; m++)
                    for (int n = 0; n < N; n++) {
                        double ref = 0;
                        for (int k = 0; k < 64; k++) {
                            const float a = mode == 0 ? fA[(r + m) * 64 + k] : fA[(r + k) * 128 + m];
                            ref += (double)a * fB[n * 64 + k];
                        }
                        maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
                    }
                if (maxerr > 0) bad_shifts++;
                printf("mode %d (%s) base_offset=%s shift r=%2d : max|err| = %g\n", mode, mode ? "MN-major, K shift" : "K-major, M shift",
                       use_base ? "(addr>>7)&7" : "0", r, maxerr);
            }
            printf("==> mode %d base %d: %d of 16 shifts wrong\n", mode, use_base, bad_shifts);
        }
    return 0;
}
