// tc_gemm.cu -- the tensor-core core of the hot path: one persistent, warp-specialised
// tcgen05 GEMM whose operand loaders understand convolution (TMA im2col mode over channels-last
// activations) as well as plain 2-D tiles.  The same kernel serves
//   conv forward            (A = im2col(X) K-major, B = repacked W K-major, epilogue bias+ReLU)
//   conv backward-data s=1  (A = im2col(dY) with pad k-1-p K-major, B = flipped W^T K-major)
//   conv backward-weight    (A = im2col(X) MN-major, B = dY MN-major, split-K FP32 partials)
//   inner product f/d/w     (plain 2-D tiles, K- or MN-major)
// Paper: the conv layer's forward/backward contract P:156 (Sec. 3.2); formulas S:145.
//
// Roles (256 threads, 1 CTA per SM, persistent over work units):
//   warp 0 lane 0 : TMA producer          (smem ring: full/empty mbarriers)
//   warp 1 lane 0 : tcgen05.mma issuer    (accumulator double buffer in TMEM)
//   warp 2        : TMEM allocator
//   warps 4..7    : epilogue (tcgen05.ld -> bias/ReLU/beta -> global), TMEM lanes 32*(w-4)..
// CG = 2 runs the CTA-pair form: a cluster of 2 CTAs computes a 256-row tile with
// tcgen05.mma.cta_group::2 (issued by the leader CTA); each CTA stages its own 128 rows of A and
// half of the B tile, so per-SM shared-memory operand traffic for B is halved.  TMA completions of
// both CTAs land on the leader's full barrier; MMA commits are multicast to both CTAs; both
// epilogues release the accumulator on the leader's barrier.
#include "internal.h"
#include "ptx.cuh"
#include "epilogue.cuh"

#include <cuda_bf16.h>

#include <cstdio>
#include <mutex>

namespace cb {

constexpr int BM = 128;
constexpr int A_STAGE_BYTES = 16384;   // 128 rows x 128 B
constexpr int SMEM_ALIGN = 1024;

constexpr int EPI_STAGE_BYTES = 4 * 2 * 4096;   // TMA-store staging: 4 epilogue warps x 2 buffers
constexpr int SGD_STAGE_BYTES = 4 * 2 * 10240;  // fused SGD: 4 warps x 2 buffers x (W 4 KB + v 4 KB + W_bf16 2 KB)
constexpr int ROWS_STAGE_BYTES = 4 * 32 * 17 * 16;   // row-staged epilogue: 4 epilogue warps x 8.5 KB
size_t tc_smem_bytes(const TcArgs& a) {
    const int macc = a.macc > 1 ? a.macc : 1;
    return (size_t)a.stages * (macc * A_STAGE_BYTES + a.b_stage_bytes) + 256 /*barriers*/ + 2 * 256 * 4 /*bias*/ +
           SMEM_ALIGN + 1024 + (a.tma_store ? (a.sgd ? SGD_STAGE_BYTES : EPI_STAGE_BYTES) : 0) +
           (a.rows_epi ? ROWS_STAGE_BYTES : 0);
}

template <int ESZ, int AMODE, int BMODE, int EPI, int CG>
__global__ void __launch_bounds__(256, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, const __grid_constant__ CUtensorMap mapV,
                   const __grid_constant__ CUtensorMap mapWb, const TcArgs args) {
    constexpr int CH = 128 / ESZ;          // elements per 128-byte row (= K per stage, = MN per chunk)
    constexpr int UMMA_K = 32 / ESZ;       // K per tcgen05.mma
    constexpr int KSTEPS = CH / UMMA_K;    // MMAs per stage (4)
    constexpr int TM = BM * CG;            // rows of a work tile
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + SMEM_ALIGN - 1) &
                                               ~uintptr_t(SMEM_ALIGN - 1));
    const int stages = args.stages;
    const int macc = args.macc > 1 ? args.macc : 1;                    // accumulators (M tiles) per unit
    const int mt_real = args.m_tiles_real > 0 ? args.m_tiles_real : args.m_tiles * macc;
    const int a_bytes = macc * A_STAGE_BYTES;
    const int stage_bytes = a_bytes + args.b_stage_bytes;
    const int nslots = 2 * macc * args.acc_stride <= args.tmem_cols ? 2 : 1;   // TMEM accumulator buffers
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + stages;
    uint64_t* tfull = empty + stages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    float* sbias = reinterpret_cast<float*>(smem + stages * stage_bytes + 256);   // [2][256]
    uint8_t* epi_stage = smem + ((stages * stage_bytes + 256 + 2048 + 1023) & ~1023);   // TMA-store buffers
    uint8_t* rows_stage = epi_stage + (args.tma_store ? (args.sgd ? SGD_STAGE_BYTES : EPI_STAGE_BYTES) : 0);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
        for (int i = 0; i < stages; i++) {
            mbar_init(&full[i], CG);          // leader: own arrive(+tx) and the peer's arrive
            mbar_init(&empty[i], 1);          // one (multicast) MMA commit
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128 * CG);  // every epilogue thread of the pair
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        if (CG == 2) tmem_alloc_cg2(tmem_holder, args.tmem_cols);
        else tmem_alloc(tmem_holder, args.tmem_cols);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    pdl_wait_and_trigger();

    if (warp == 0 && lane == 0) {
        // ===================== TMA producer (both CTAs) =====================
        int stage = 0;
        uint32_t phase = 0;
        const int bn_cta = args.BN / CG;                            // B rows (K-major) staged by this CTA
        for (int u = cid; u < args.units; u += ncl) {
            int t = u;
            const int n_tile = t % args.n_tiles; t /= args.n_tiles;
            const int m_tile = t % args.m_tiles; t /= args.m_tiles;
            const int g = t % args.groups;
            const int split = t / args.groups;
            const int kb0 = split * args.kb_per_split;
            const int kb1 = min(args.kblocks, kb0 + args.kb_per_split);
            const int nacc = min(macc, mt_real - m_tile * macc);         // M tiles present in this unit
            // bytes landing in THIS CTA per stage
            const uint32_t tx = (uint32_t)(nacc * A_STAGE_BYTES + args.b_stage_bytes);
            const int m0 = m_tile * TM + (int)rank * BM;   // first row staged by this CTA
            int an = 0, ay = 0, ax = 0;
            if (AMODE == A_IM2COL_K) {
                an = m0 / args.a_P;
                const int r = m0 - an * args.a_P;
                ay = r / args.a_OW;
                ax = r - ay * args.a_OW;
            }
            // im2col K order: kb = (i*kw + j)*cblocks + cbk, tracked incrementally (no per-stage division)
            int cbk = 0, ti = 0, tj = 0;
            if (AMODE == A_IM2COL_K) {
                const int tap0 = kb0 / args.a_cblocks;
                cbk = kb0 - tap0 * args.a_cblocks;
                ti = tap0 / args.a_kw;
                tj = tap0 - ti * args.a_kw;
            }
            for (int kb = kb0; kb < kb1; kb++) {
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = smem + stage * stage_bytes;
                uint8_t* sb = sa + a_bytes;
                if (CG == 1 || leader) mbar_arrive_expect_tx(&full[stage], tx * CG);
                else mbar_arrive_cluster(mapa_shared(smem_u32(&full[stage]), 0));
                // ---- A
                if (AMODE == A_TILED_K) {
                    if (CG == 2) tma_load_2d_cg2(sa, &mapA, &full[stage], kb * CH, g * args.a_row_g + m0);
                    else tma_load_2d(sa, &mapA, &full[stage], kb * CH, g * args.a_row_g + m0);
                } else if (AMODE == A_IM2COL_K) {
                    if (CG == 2)
                        tma_load_im2col_4d_cg2(sa, &mapA, &full[stage], g * args.a_cpg + cbk * CH, ax - args.a_pad_w,
                                               ay - args.a_pad_h, an, (uint16_t)tj, (uint16_t)ti);
                    else
                        tma_load_im2col_4d(sa, &mapA, &full[stage], g * args.a_cpg + cbk * CH, ax - args.a_pad_w,
                                           ay - args.a_pad_h, an, (uint16_t)tj, (uint16_t)ti);
                    if (++cbk == args.a_cblocks) {
                        cbk = 0;
                        if (++tj == args.a_kw) { tj = 0; ++ti; }
                    }
                } else if (AMODE == A_IM2COL_MN) {
                    const int p0 = kb * CH;   // first pixel of this reduction block
                    const int n0 = p0 / args.a_P;
                    const int r = p0 - n0 * args.a_P;
                    const int y0 = r / args.a_OW, x0 = r - (r / args.a_OW) * args.a_OW;
                    for (int a = 0; a < nacc; a++) {
#pragma unroll
                        for (int q = 0; q < ESZ; q++) {   // 128 rows of M = ESZ chunks of CH
                            int chunk = ((m_tile * macc + a) * CG + (int)rank) * ESZ + q;
                            if (chunk >= args.a_nchunks_total) chunk = args.a_nchunks_total - 1;  // rows discarded
                            const int tap = chunk / args.a_cblocks, cbk = chunk - tap * args.a_cblocks;
                            const int i = tap / args.a_kw, j = tap - i * args.a_kw;
                            tma_load_im2col_4d(sa + a * A_STAGE_BYTES + q * CH * 128, &mapA, &full[stage],
                                               g * args.a_cpg + cbk * CH, x0 - args.a_pad_w, y0 - args.a_pad_h, n0,
                                               (uint16_t)j, (uint16_t)i);
                        }
                    }
                } else {  // A_TILED_MN
#pragma unroll
                    for (int q = 0; q < ESZ; q++) {
                        if (CG == 2)
                            tma_load_2d_cg2(sa + q * CH * 128, &mapA, &full[stage], g * args.a_row_g + m0 + q * CH,
                                            kb * CH);
                        else
                            tma_load_2d(sa + q * CH * 128, &mapA, &full[stage], g * args.a_row_g + m0 + q * CH, kb * CH);
                    }
                }
                // ---- B
                if (BMODE == B_TILED_K) {
                    const int row = g * args.b_row_g + n_tile * args.BN + (int)rank * bn_cta;
                    if (CG == 2) tma_load_2d_cg2(sb, &mapB, &full[stage], kb * CH, row);
                    else tma_load_2d(sb, &mapB, &full[stage], kb * CH, row);
                } else {
                    // MN-major B: 64-column chunks; a CTA pair splits them (each CTA stages its half)
                    const int nch = args.b_nchunks / CG;
                    for (int q = 0; q < nch; q++) {
                        const int col = g * args.b_col_g + n_tile * args.BN + ((int)rank * nch + q) * CH;
                        if (CG == 2) tma_load_2d_cg2(sb + q * CH * 128, &mapB, &full[stage], col, kb * CH);
                        else tma_load_2d(sb + q * CH * 128, &mapB, &full[stage], col, kb * CH);
                    }
                }
                if (++stage == stages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1 && leader) {
        // ===================== MMA issuer (leader CTA, whole warp) =====================
        // The warp runs the loop convergently so descriptors stay warp-uniform (uniform registers,
        // no per-MMA register->uniform waterfall); one elected lane issues the tcgen05 ops.
        // instruction descriptor: D=f32, A/B format (bf16=1, tf32=2), majors, N>>3, M>>4
        const uint32_t fmt = (ESZ == 2) ? 1u : 2u;
        const uint32_t a_mn = (AMODE == A_IM2COL_MN || AMODE == A_TILED_MN) ? 1u : 0u;
        const uint32_t b_mn = (BMODE == B_TILED_MN) ? 1u : 0u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (a_mn << 15) | (b_mn << 16) |
                               ((uint32_t)(args.BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
        // per-K-step descriptor advance (start address field is in 16-byte units):
        // K-major: 32 bytes along the 128-byte row; MN-major: UMMA_K rows of 128 bytes
        const uint64_t a_step = a_mn ? (uint64_t)(UMMA_K * 128 / 16) : 2ull;
        const uint64_t b_step = b_mn ? (uint64_t)(UMMA_K * 128 / 16) : 2ull;
        const uint32_t a_lbo = a_mn ? CH * 128 : 16, b_lbo = b_mn ? CH * 128 : 16;
        const uint32_t smem_base = smem_u32(smem);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        int iters = 0;
        for (int u = cid; u < args.units; u += ncl, iters++) {
            const int m_tile = (u / args.n_tiles) % args.m_tiles;
            int t = u / (args.n_tiles * args.m_tiles);
            const int split = t / args.groups;
            const int kb0 = split * args.kb_per_split;
            const int kb1 = min(args.kblocks, kb0 + args.kb_per_split);
            const int nacc = min(macc, mt_real - m_tile * macc);
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * macc * args.acc_stride;
            for (int kb = kb0; kb < kb1; kb++) {
                if (args.spin) mbar_wait_spin(&full[stage], phase);
                else mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t sa = smem_base + stage * stage_bytes;
                const uint64_t bd0 = operand_desc<ESZ>(sa + a_bytes, b_lbo, b_mn);
                if (elect_one()) {
                    for (int a = 0; a < nacc; a++) {
                        const uint64_t ad0 = operand_desc<ESZ>(sa + a * A_STAGE_BYTES, a_lbo, a_mn);
                        const uint32_t dt = d_tmem + a * args.acc_stride;
#pragma unroll
                        for (int k = 0; k < KSTEPS; k++) {
                            const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
                            if (CG == 2) umma_cg2<ESZ>(dt, ad0 + k * a_step, bd0 + k * b_step, idesc, accum);
                            else umma<ESZ>(dt, ad0 + k * a_step, bd0 + k * b_step, idesc, accum);
                        }
                    }
                    if (CG == 2) umma_commit_cg2(&empty[stage]);
                    else umma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == stages) { stage = 0; phase ^= 1; }
            }
            if (elect_one()) {
                if (CG == 2) umma_commit_cg2(&tfull[acc]);
                else umma_commit(&tfull[acc]);
            }
            __syncwarp();
            if (++acc == nslots) { acc = 0; acc_phase ^= 1; }
        }
        // the peer's epilogue arrives remotely on our tempty barriers: drain the last two phases
        // before the pair tears down
        if (CG == 2 && iters > 0) {
            if (nslots == 2) {
                for (int j = iters - 2; j < iters; j++)
                    if (j >= 0) mbar_wait(&tempty[j & 1], (uint32_t)((j >> 1) & 1));
            } else {
                mbar_wait(&tempty[0], (uint32_t)((iters - 1) & 1));
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs) =====================
        const int q = warp - 4;
        const int row = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
        int tbuf = 0;
        // the whole bias vector (groups x N <= 512 columns, whole N tiles) staged once per kernel
        // instead of each unit's columns behind a barrier; a unit reads its columns at offset cbase
        const int nbias = args.groups * args.N;
        const bool bias_const = args.bias && EPI != EPI_SGD && nbias <= 512 && args.N % args.BN == 0 &&
                                args.col_g == args.N;
        if (bias_const) {
            for (int c = row; c < nbias; c += 128) sbias[c] = args.bias[c];
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        for (int u = cid; u < args.units; u += ncl) {
            int t = u;
            const int n_tile = t % args.n_tiles; t /= args.n_tiles;
            const int m_tile = t % args.m_tiles; t /= args.m_tiles;
            const int g = t % args.groups;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * macc * args.acc_stride;
            if (EPI == EPI_PARTIAL) {
                const int split = t / args.groups;
                const int nacc = min(macc, mt_real - m_tile * macc);
                for (int a = 0; a < nacc; a++) {
                    // partial slot of the one-tile unit (split, g, m_tile*macc + a, n_tile)
                    const size_t vu = (((size_t)split * args.groups + g) * mt_real + (m_tile * macc + a)) *
                                          args.n_tiles + n_tile;
                    float* dst = args.partial + vu * args.BN * TM + (int)rank * BM + row;
                    for (int c0 = 0; c0 < args.BN; c0 += 32) {
                        const bool two = c0 + 16 < args.BN;
                        uint32_t v0[16], v1[16];
                        tmem_ld16(taddr + a * args.acc_stride + c0, v0);
                        if (two) tmem_ld16(taddr + a * args.acc_stride + c0 + 16, v1);
                        tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 16; j++) dst[(size_t)(c0 + j) * TM] = __uint_as_float(v0[j]);
                        if (two) {
#pragma unroll
                            for (int j = 0; j < 16; j++) dst[(size_t)(c0 + 16 + j) * TM] = __uint_as_float(v1[j]);
                        }
                    }
                }
            } else {
                const int m = m_tile * TM + (int)rank * BM + row;
                const bool row_ok = m < args.M;
                const int img = m / args.P, pix = m - img * args.P;
                const long long rbase = (long long)img * args.s_n + (long long)pix * args.s_p;
                const int col0 = n_tile * args.BN;
                const int cbase = g * args.col_g + col0;   // output channel of tile column 0
                // stage this tile's bias once (double-buffered by accumulator: a warp can be at most
                // one tile ahead of the slowest epilogue warp)
                float* bs = bias_const ? sbias + cbase : sbias + acc * 256;
                if (args.bias && !bias_const) {
                    for (int c = row; c < args.BN; c += 128) bs[c] = (col0 + c < args.N) ? args.bias[cbase + c] : 0.f;
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                }
                // (the fused-update epilogue is its own template instance: its registers would
                // otherwise stop the 48-register update kernel co-residing beside every GEMM CTA)
                if constexpr (EPI == EPI_SGD) {
                    epi_sgd_tma(args, &mapC, &mapV, &mapWb, taddr, m_tile * TM + (int)rank * BM + q * 32, col0, cbase,
                                epi_stage + q * 20480, tbuf, lane);
                } else if (args.tma_store) {
                    epi_store_tma(args, &mapC, taddr, m_tile * TM + (int)rank * BM + q * 32, col0, cbase, bs,
                                  epi_stage + q * 8192, tbuf, lane);
                } else if (args.rows_epi) {
                    epi_store_rows(args, taddr, row_ok, rbase, col0, cbase, bs, rows_stage + q * (32 * 17 * 16), lane);
                } else {
                    epi_store_strided(args, taddr, row_ok, rbase, col0, cbase, bs);
                }
            }
            tc_fence_before();
            if (CG == 2) mbar_arrive_cluster(tempty_leader + (uint32_t)acc * 8u);
            else mbar_arrive(&tempty[acc]);
            if (++acc == nslots) { acc = 0; acc_phase ^= 1; }
        }
        if (args.tma_store && lane == 0) tma_store_wait_all();
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_cg2(tmem_base, args.tmem_cols);
        else tmem_dealloc(tmem_base, args.tmem_cols);
    }
}

// ------------------------------------------------------------------ host side
int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int g_pdl = 0;   // CAFFE_TUNE_PDL

template <int ESZ, int AM, int BMd, int EP, int CG>
static cudaError_t launch_one(const TcLaunch& L, cudaStream_t s) {
    auto kern = tc_gemm_kernel<ESZ, AM, BMd, EP, CG>;
    const size_t smem = tc_smem_bytes(L.args);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_tc(kern, L.grid, 256, smem, s, CG, L.mapA, L.mapB, L.mapC, L.mapV, L.mapWb, L.args);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

#define TC_CASE(E, A, B, P, G)                                                                   \
    if (L.esz == E && L.amode == A && L.bmode == B && L.epi == P && L.cg == G) return launch_one<E, A, B, P, G>(L, s);

cudaError_t tc_launch(const TcLaunch& L, cudaStream_t s) {
    TC_CASE(2, A_IM2COL_K, B_TILED_K, EPI_STRIDED, 1)
    TC_CASE(2, A_IM2COL_K, B_TILED_K, EPI_STRIDED, 2)
    TC_CASE(2, A_IM2COL_MN, B_TILED_MN, EPI_PARTIAL, 1)
    TC_CASE(2, A_TILED_K, B_TILED_K, EPI_STRIDED, 1)
    TC_CASE(2, A_TILED_K, B_TILED_K, EPI_STRIDED, 2)
    TC_CASE(2, A_TILED_K, B_TILED_MN, EPI_STRIDED, 1)
    TC_CASE(2, A_TILED_K, B_TILED_K, EPI_PARTIAL, 1)
    TC_CASE(2, A_TILED_K, B_TILED_K, EPI_PARTIAL, 2)
    TC_CASE(2, A_TILED_K, B_TILED_MN, EPI_PARTIAL, 1)
    TC_CASE(2, A_TILED_K, B_TILED_MN, EPI_PARTIAL, 2)
    TC_CASE(2, A_TILED_K, B_TILED_MN, EPI_STRIDED, 2)
    TC_CASE(2, A_TILED_MN, B_TILED_MN, EPI_STRIDED, 2)
    TC_CASE(2, A_TILED_MN, B_TILED_MN, EPI_SGD, 2)
    TC_CASE(2, A_TILED_MN, B_TILED_MN, EPI_SGD, 1)
    TC_CASE(4, A_TILED_K, B_TILED_K, EPI_PARTIAL, 1)
    TC_CASE(4, A_IM2COL_MN, B_TILED_MN, EPI_PARTIAL, 1)
    TC_CASE(4, A_TILED_K, B_TILED_MN, EPI_STRIDED, 1)
    TC_CASE(4, A_TILED_K, B_TILED_MN, EPI_PARTIAL, 1)
    TC_CASE(4, A_TILED_MN, B_TILED_MN, EPI_STRIDED, 1)
    TC_CASE(2, A_TILED_MN, B_TILED_MN, EPI_STRIDED, 1)
    TC_CASE(4, A_IM2COL_K, B_TILED_K, EPI_STRIDED, 1)
    TC_CASE(4, A_TILED_K, B_TILED_K, EPI_STRIDED, 1)
    return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ TMA descriptor encoding
typedef CUresult (*PFN_tiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_im2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_tiled g_tiled = nullptr;
static PFN_im2col g_im2col = nullptr;

static bool resolve() {
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_tiled = reinterpret_cast<PFN_tiled>(p);
        p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_im2col = reinterpret_cast<PFN_im2col>(p);
    });
    return g_tiled && g_im2col;
}

bool encode_tiled_2d(CUtensorMap* m, int esz, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                     uint32_t box_inner, uint32_t box_outer, bool mn_tf32) {
    if (!resolve()) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_tiled(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                         const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         mn_tf32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_store_2d(CUtensorMap* m, int esz, const void* base, uint64_t cols, uint64_t rows, uint64_t ld) {
    if (!resolve()) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * esz};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_tiled(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                         const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// channels-last activation [N][H][W][C] as a 4-D tiled map; box (box_c channels, box_w, box_h, 1)
bool encode_tiled_4d(CUtensorMap* m, int esz, const void* base, int C, int W, int H, int N, uint32_t box_c,
                     uint32_t box_w, uint32_t box_h) {
    if (!resolve()) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * esz, (cuuint64_t)C * W * esz, (cuuint64_t)C * W * H * esz};
    cuuint32_t box[4] = {box_c, box_w, box_h, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = g_tiled(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                         const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_store_2d_bf16_32(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld) {
    if (!resolve()) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_store_4d(CUtensorMap* m, int esz, const void* base, int C, int W, int H, int N, long long s_p,
                     long long s_n, uint32_t box_c, uint32_t box_w, uint32_t box_h, int swizzle_bytes) {
    if (!resolve()) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)(s_p * esz), (cuuint64_t)(s_p * W * esz), (cuuint64_t)(s_n * esz)};
    cuuint32_t box[4] = {box_c, box_w, box_h, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = g_tiled(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                         const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_im2col_4d(CUtensorMap* m, int esz, const void* base, int C, int W, int H, int N, int pad_lo_w,
                      int pad_lo_h, int up_w, int up_h, uint32_t channels, uint32_t pixels, bool mn_tf32) {
    if (!resolve()) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)C * esz, (cuuint64_t)C * W * esz, (cuuint64_t)C * W * H * esz};
    int lower[2] = {-pad_lo_w, -pad_lo_h};
    int upper[2] = {up_w, up_h};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = g_im2col(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                          const_cast<void*>(base), dims, strides, lower, upper, channels, pixels, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          mn_tf32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace cb
