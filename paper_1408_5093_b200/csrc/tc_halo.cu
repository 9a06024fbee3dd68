// tc_halo.cu -- stride-1 convolution as a halo-tiled implicit GEMM on tcgen05.
//
// The im2col formulation (tc_gemm.cu, A_IM2COL_K) stages a 128-pixel x 64-channel A tile per filter
// tap, so every activation byte crosses L2->SM once per tap (25x for 5x5) and the passes run at the
// chip's TMA throughput.  Here a work tile is halo_th whole output rows (padded to halo_wt =
// OW + kw - 1 columns) of one image; its input window -- (halo_th + kh - 1) rows x halo_wt columns x
// 64 channels -- is loaded ONCE per channel block with a 4-D tiled TMA (zero fill supplies the
// padding), and tap (i, j) feeds tcgen05.mma the same shared-memory tile through a descriptor whose
// start is moved by (i*halo_wt + j) rows of 128 bytes.  Accumulator row m = r*halo_wt + x is output
// pixel (y0 + r, x); columns x >= OW are discarded by the epilogue.  (The 128-byte swizzle is a
// function of the absolute shared-memory address, so row-shifted descriptors with base offset 0
// read exactly the rows they name -- checked by tools/desc_probe.cu.)
//
// Used for the conv forward (A = X, B = repacked W) and the stride-1 data gradient (A = dY with pad
// k-1-p, B = flipped W^T).  Paper: the layer contract P:156; formulas S:145.
//
// Roles: warp 0 lane 0 TMA producer (A ring of halo stages + B ring of per-tap weight tiles),
// warp 1 MMA issuer (leader CTA; whole warp, one elected lane issues), warp 2 TMEM allocator,
// warps 4..7 epilogue.  A unit holds `macc` tiles per CTA (accumulators) that share every B tile;
// CG = 2 pairs two SMs (cta_group::2): each CTA stages its own tiles and half of each B tile.
#include "internal.h"
#include "ptx.cuh"
#include "epilogue.cuh"

#include <cuda_bf16.h>

namespace cb {

constexpr int HALO_SMEM_ALIGN = 1024;
int g_halo_fast_epi = 1;   // CAFFE_TUNE_HALO_FAST_EPI
int g_halo_coal = 1;       // CAFFE_TUNE_HALO_COALESCE
int g_halo_tma_store = 0;   // CAFFE_TUNE_HALO_TMA_STORE (off: measured no gain for conv1, conv2 fwd 92 -> 106 us)

int g_halo_epi_groups = 0;   // CAFFE_TUNE_HALO_EPI_GROUPS (0 = automatic)

// per-CTA staging of the coalesced specialised epilogue: 4 warps per epilogue group
size_t halo_coal_bytes(const TcArgs& a) {
    const int ng = a.epi_groups >= 3 ? a.epi_groups : 2;
    const int epc = a.BN / ng;
    return (size_t)4 * ng * 32 * ((epc / 8) | 1) * 16;
}

size_t tc_halo_smem_bytes(const TcArgs& a) {
    const int macc = a.macc > 1 ? a.macc : 1;
    return (size_t)a.a_stages * (a.a_merge ? 1 : macc) * a.halo_slot + (size_t)a.stages * a.b_stage_bytes + 512 /*barriers*/ +
           2 * 256 * 4 /*bias*/ + HALO_SMEM_ALIGN + (a.rows_epi ? 4 * 32 * 17 * 16 : 0) +
           (a.tma_store ? (size_t)macc * a.st_tile_bytes + 1024 : 0) + (a.epi_coal ? halo_coal_bytes(a) + 1024 : 0);
}

// KS: 16-channel K steps issued per 64-channel block (4; 3 when the only block holds 48 real
// channels -- conv1 after space-to-depth, conv2 per group -- so the zero padding is not multiplied)
// EPC > 0: the specialised channels-last BF16 epilogue (epi_store_bf16_rowseg), each of the NEG
// epilogue groups (4 warps each) writing EPC = BN/NEG columns
template <int CG, int MACC, int KS, int EPC, int BT, int NEG = 2>
__global__ void __launch_bounds__(128 + 128 * NEG, 1)
    tc_halo_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, const TcArgs args) {
    constexpr int CH = 64;                 // bf16 channels per 128-byte row
    constexpr int KSTEPS = KS;             // K = 16 per tcgen05.mma
    constexpr int TM = 128 * CG;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + HALO_SMEM_ALIGN - 1) &
                                               ~uintptr_t(HALO_SMEM_ALIGN - 1));
    constexpr int macc = MACC;             // accumulators (tiles) per CTA per unit
    const int a_stages = args.a_stages, b_stages = args.stages;
    const int slot = args.halo_slot;
    // a_merge: the MACC tiles of a CTA are consecutive row blocks of one image and share ONE staged
    // window (accumulator a reads it shifted by a*halo_th*halo_wt rows)
    const bool merge = args.a_merge != 0;
    const int a_stage_bytes = merge ? slot : macc * slot;
    const uint32_t acc_rows_b = (uint32_t)(args.halo_th * args.halo_wt * 128);
    uint8_t* a_ring = smem;
    uint8_t* b_ring = smem + a_stages * a_stage_bytes;
    uint64_t* fullA = reinterpret_cast<uint64_t*>(b_ring + b_stages * args.b_stage_bytes);
    uint64_t* emptyA = fullA + a_stages;
    uint64_t* fullB = emptyA + a_stages;
    uint64_t* emptyB = fullB + b_stages;
    uint64_t* tfull = emptyB + b_stages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    float* sbias = reinterpret_cast<float*>(b_ring + b_stages * args.b_stage_bytes + 512);   // [2][256]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
    const int nslots = 2 * macc * args.acc_stride <= args.tmem_cols ? 2 : 1;
    const int taps = args.halo_kh * args.a_kw;
    const int cblocks = args.a_cblocks;
    const int tiles_per_unit = macc * CG;
    const int tgroups = (args.total_tiles + tiles_per_unit - 1) / tiles_per_unit;
    const int units = args.groups * args.n_tiles * tgroups;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
        for (int i = 0; i < a_stages; i++) { mbar_init(&fullA[i], CG); mbar_init(&emptyA[i], 1); }
        for (int i = 0; i < b_stages; i++) { mbar_init(&fullB[i], CG); mbar_init(&emptyB[i], 1); }
        for (int i = 0; i < 2; i++) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128 * NEG * CG); }
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
        const uint32_t txA = args.stk ? (uint32_t)(macc * args.stk_nb * args.stk_wt * 128)
                                      : (uint32_t)((merge ? 1 : macc) * args.halo_rows * args.halo_wt * 128);
        const uint32_t txB = (uint32_t)args.b_stage_bytes;
        const int bn_cta = args.BN / CG;
        int sa = 0, sb = 0;
        uint32_t pa = 0, pb = 0;
        if (args.b_resident) {
            // every (tap, channel block) weight tile once, into its own slot, on one barrier
            const int nb = taps * cblocks;
            if (CG == 1 || leader) mbar_arrive_expect_tx(&fullB[0], txB * CG * nb);
            else mbar_arrive_cluster(mapa_shared(smem_u32(&fullB[0]), 0));
            for (int kb = 0; kb < nb; kb++) {
                uint8_t* dst = b_ring + kb * args.b_stage_bytes;
                if (CG == 2) tma_load_2d_cg2(dst, &mapB, &fullB[0], kb * CH, (int)rank * bn_cta);
                else tma_load_2d(dst, &mapB, &fullB[0], kb * CH, (int)rank * bn_cta);
            }
        }
        for (int u = cid; u < units; u += ncl) {
            int t = u;
            const int n_tile = t % args.n_tiles; t /= args.n_tiles;
            const int tg = t % tgroups;
            const int g = t / tgroups;
            for (int cb = 0; cb < cblocks; cb++) {
                mbar_wait(&emptyA[sa], pa ^ 1);
                if (CG == 1 || leader) mbar_arrive_expect_tx(&fullA[sa], txA * CG);
                else mbar_arrive_cluster(mapa_shared(smem_u32(&fullA[sa]), 0));
                for (int a = 0; a < (merge ? 1 : macc); a++) {
                    int tile = tg * tiles_per_unit + (merge ? (int)rank * macc : a * CG + (int)rank);
                    if (tile >= args.total_tiles) tile = args.total_tiles - 1;   // rows discarded
                    uint8_t* dst = a_ring + sa * a_stage_bytes + a * slot;
                    const int c = g * args.a_cpg + cb * CH;
                    if (args.stk) {
                        // one-row boxes: stacked row b (image b / hs, padded row b % hs) at shared row
                        // stk_off - (m0 - b0*wt) + q*wt, so the tile's first pixel is at row stk_off
                        const int m0 = tile * 128;
                        const int b0 = m0 / args.stk_wt;
                        int img = b0 / args.stk_hs, lb = b0 - img * args.stk_hs;
                        uint8_t* d = dst + (args.stk_off - (m0 - b0 * args.stk_wt)) * 128;
                        for (int q = 0; q < args.stk_nb; q++) {
                            if (CG == 2) tma_load_4d_cg2(d, &mapA, &fullA[sa], c, -args.a_pad_w, lb - args.a_pad_h, img);
                            else tma_load_4d(d, &mapA, &fullA[sa], c, -args.a_pad_w, lb - args.a_pad_h, img);
                            d += args.stk_wt * 128;
                            if (++lb == args.stk_hs) { lb = 0; img++; }
                        }
                        continue;
                    }
                    const int n = tile / args.tiles_per_img;
                    const int y0 = (tile - n * args.tiles_per_img) * args.halo_th;
                    if (CG == 2) tma_load_4d_cg2(dst, &mapA, &fullA[sa], c, -args.a_pad_w, y0 - args.a_pad_h, n);
                    else tma_load_4d(dst, &mapA, &fullA[sa], c, -args.a_pad_w, y0 - args.a_pad_h, n);
                }
                if (++sa == a_stages) { sa = 0; pa ^= 1; }
                if (args.b_resident) continue;
                // BT weight tiles (taps) per B stage; BT divides the tap count (host)
                for (int tap = 0; tap < taps; tap += BT) {
                    mbar_wait(&emptyB[sb], pb ^ 1);
                    if (CG == 1 || leader) mbar_arrive_expect_tx(&fullB[sb], txB * CG);
                    else mbar_arrive_cluster(mapa_shared(smem_u32(&fullB[sb]), 0));
                    const int row = g * args.b_row_g + n_tile * args.BN + (int)rank * bn_cta;
#pragma unroll
                    for (int j = 0; j < BT; j++) {
                        const int kb = (tap + j) * cblocks + cb;
                        uint8_t* dst = b_ring + sb * args.b_stage_bytes + j * (args.b_stage_bytes / BT);
                        if (CG == 2) tma_load_2d_cg2(dst, &mapB, &fullB[sb], kb * CH, row);
                        else tma_load_2d(dst, &mapB, &fullB[sb], kb * CH, row);
                    }
                    if (++sb == b_stages) { sb = 0; pb ^= 1; }
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ===================== MMA issuer (leader CTA, whole warp) =====================
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(args.BN >> 3) << 17) |
                               ((uint32_t)(TM >> 4) << 24);
        const uint32_t a_base = smem_u32(a_ring), b_base = smem_u32(b_ring);
        int sa = 0, sb = 0, acc = 0, iters = 0;
        uint32_t pa = 0, pb = 0, acc_phase = 0;
        if (args.b_resident) {
            mbar_wait(&fullB[0], 0);
            tc_fence_after();
        }
        for (int u = cid; u < units; u += ncl, iters++) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * macc * args.acc_stride;
            for (int cb = 0; cb < cblocks; cb++) {
                mbar_wait(&fullA[sa], pa);
                tc_fence_after();
                const uint32_t sa_addr = a_base + sa * a_stage_bytes;
                // tap (i, j) reads the staged window shifted by i*halo_wt + j rows (no division in
                // the issue loop: the MMA warp's instruction latency bounds small-N tiles); stacked
                // tiles start at row stk_off of their slot
                uint32_t shift = (uint32_t)args.stk_off * 128u;
                int tj = 0;
                const uint32_t row_skip = (uint32_t)(args.halo_wt - args.a_kw + 1) * 128u;
                if constexpr (BT > 1) {
                    // BT taps per B stage: one barrier wait and one commit per BT x MACC x KSTEPS MMAs
                    // (the issue loop's own instructions bound the short-N tiles)
                    const uint32_t b_tile = (uint32_t)(args.b_stage_bytes / BT);
                    for (int tap = 0; tap < taps; tap += BT) {
                        mbar_wait(&fullB[sb], pb);
                        tc_fence_after();
                        const uint64_t bs0 = smem_desc_sw128(b_base + (uint32_t)sb * (uint32_t)args.b_stage_bytes, 16, 1024);
                        if (elect_one()) {
                            uint32_t sh = shift;
                            int tjj = tj;
#pragma unroll
                            for (int j = 0; j < BT; j++) {
                                const uint64_t bd0 = bs0 + (uint64_t)((j * b_tile) >> 4);
#pragma unroll
                                for (int a = 0; a < MACC; a++) {
                                    const uint64_t ad0 =
                                        smem_desc_sw128(sa_addr + (merge ? a * acc_rows_b : a * slot) + sh, 16, 1024);
                                    const uint32_t dt = d_tmem + a * args.acc_stride;
#pragma unroll
                                    for (int k = 0; k < KSTEPS; k++) {
                                        const uint32_t accum = (cb > 0 || tap + j > 0 || k > 0) ? 1u : 0u;
                                        if (CG == 2) umma_cg2<2>(dt, ad0 + 2 * k, bd0 + 2 * k, idesc, accum);
                                        else umma<2>(dt, ad0 + 2 * k, bd0 + 2 * k, idesc, accum);
                                    }
                                }
                                if (++tjj == args.a_kw) { tjj = 0; sh += row_skip; }
                                else sh += 128u;
                            }
                            if (CG == 2) umma_commit_cg2(&emptyB[sb]);
                            else umma_commit(&emptyB[sb]);
                        }
                        __syncwarp();
                        if (++sb == b_stages) { sb = 0; pb ^= 1; }
#pragma unroll
                        for (int j = 0; j < BT; j++) {
                            if (++tj == args.a_kw) { tj = 0; shift += row_skip; }
                            else shift += 128u;
                        }
                    }
                } else
                for (int tap = 0; tap < taps; tap++) {
                    const bool bres = args.b_resident != 0;
                    if (!bres) {
                        mbar_wait(&fullB[sb], pb);
                        tc_fence_after();
                    }
                    const uint32_t bslot = bres ? (uint32_t)(tap * cblocks + cb) : (uint32_t)sb;
                    const uint64_t bd0 = smem_desc_sw128(b_base + bslot * args.b_stage_bytes, 16, 1024);
                    if (elect_one()) {
#pragma unroll
                        for (int a = 0; a < MACC; a++) {
                            const uint64_t ad0 =
                                smem_desc_sw128(sa_addr + (merge ? a * acc_rows_b : a * slot) + shift, 16, 1024);
                            const uint32_t dt = d_tmem + a * args.acc_stride;
#pragma unroll
                            for (int k = 0; k < KSTEPS; k++) {
                                const uint32_t accum = (cb > 0 || tap > 0 || k > 0) ? 1u : 0u;
                                if (CG == 2) umma_cg2<2>(dt, ad0 + 2 * k, bd0 + 2 * k, idesc, accum);
                                else umma<2>(dt, ad0 + 2 * k, bd0 + 2 * k, idesc, accum);
                            }
                        }
                        if (!bres) {
                            if (CG == 2) umma_commit_cg2(&emptyB[sb]);
                            else umma_commit(&emptyB[sb]);
                        }
                    }
                    __syncwarp();
                    if (!bres && ++sb == b_stages) { sb = 0; pb ^= 1; }
                    if (++tj == args.a_kw) { tj = 0; shift += row_skip; }
                    else shift += 128u;
                }
                if (elect_one()) {
                    if (CG == 2) umma_commit_cg2(&emptyA[sa]);
                    else umma_commit(&emptyA[sa]);
                }
                __syncwarp();
                if (++sa == a_stages) { sa = 0; pa ^= 1; }
            }
            if (elect_one()) {
                if (CG == 2) umma_commit_cg2(&tfull[acc]);
                else umma_commit(&tfull[acc]);
            }
            __syncwarp();
            if (++acc == nslots) { acc = 0; acc_phase ^= 1; }
        }
        if (CG == 2 && iters > 0) {   // the peer's epilogue arrives remotely on our tempty barriers
            if (nslots == 2) {
                for (int j = iters - 2; j < iters; j++)
                    if (j >= 0) mbar_wait(&tempty[j & 1], (uint32_t)((j >> 1) & 1));
            } else {
                mbar_wait(&tempty[0], (uint32_t)((iters - 1) & 1));
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs): NEG groups of 4 warps =====================
        // Group e (warps 4-7, 8-11, ...) writes columns [e*half, ...) of the tiles; every group reads
        // the same TMEM lanes (warp % 4 selects the lane quadrant).  Several warps per SM
        // sub-partition hide the TMEM-load and store latency of the epilogue, which bounds the
        // wide-output layers (conv1 forward: three groups).
        const int q = warp & 3;
        const int eg = (warp - 4) >> 2;
        const int row = q * 32 + lane;
        const int yy = row / args.halo_wt, xx = row - yy * args.halo_wt;
        const int half = EPC > 0 ? EPC : ((args.BN / 2) + 15) & ~15;
        const int cb_ = eg * half, ce_ = eg == NEG - 1 ? args.BN : cb_ + half;
        int acc = 0;
        uint32_t acc_phase = 0;
        const uint32_t tempty_leader = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
        // TMA-store staging (EPC > 0 && args.tma_store): one tile image per accumulator of the unit
        const bool tstore = EPC > 0 && args.tma_store != 0;
        const uint32_t stg = (smem_u32(sbias + 2 * 256) + 1023u) & ~1023u;
        const bool issuer = warp == 4 && lane == 0;
        // the whole bias vector (groups x N <= 512 columns, whole N tiles) staged once per kernel
        // instead of each unit's columns behind a group barrier (conv1 forward 75 -> 69 us); a unit
        // then reads its columns at offset cbase
        const int nbias = args.groups * args.N;
        const bool bias_const = args.bias && nbias <= 512 && args.N % args.BN == 0 && args.col_g == args.N &&
                                args.stk == 0;
        if (bias_const) {
            for (int c = row; c < nbias; c += 128) sbias[c] = args.bias[c];
            asm volatile("bar.sync %0, %1;" ::"r"(1 + NEG), "r"(128 * NEG) : "memory");
        }
        for (int u = cid; u < units; u += ncl) {
            int t = u;
            const int n_tile = t % args.n_tiles; t /= args.n_tiles;
            const int tg = t % tgroups;
            const int g = t / tgroups;
            if (tstore) {   // the previous unit's tensor stores must have finished reading the staging
                if (issuer) tma_store_wait_read0();
                asm volatile("bar.sync %0, %1;" ::"r"(1 + NEG), "r"(128 * NEG) : "memory");
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * macc * args.acc_stride;
            const int col0 = n_tile * args.BN;
            const int cbase = g * args.col_g + col0;
            float* bs = bias_const ? sbias + cbase : sbias + acc * 256;
            if (args.bias && !bias_const) {
                for (int c = cb_ + row; c < ce_; c += 128) bs[c] = (col0 + c < args.N) ? args.bias[cbase + c] : 0.f;
                asm volatile("bar.sync %0, 128;" ::"r"(1 + eg) : "memory");
            }
            for (int a = 0; a < macc; a++) {
                const int tile = tg * tiles_per_unit + (merge ? (int)rank * macc + a : a * CG + (int)rank);
                int n, y, x;
                bool row_ok;
                if (args.stk) {   // stacked pixel m = n*(hs*wt) + y*wt + x
                    const int m = tile * 128 + row;
                    const int per = args.stk_hs * args.stk_wt;
                    n = m / per;
                    const int l = m - n * per;
                    y = l / args.stk_wt;
                    x = l - y * args.stk_wt;
                    row_ok = tile < args.total_tiles && n < args.stk_nimg && y < args.out_h && x < args.out_w;
                } else {
                    n = tile / args.tiles_per_img;
                    y = (tile - n * args.tiles_per_img) * args.halo_th + yy;
                    x = xx;
                    row_ok = tile < args.total_tiles && yy < args.halo_th && y < args.out_h && xx < args.out_w;
                }
                const long long rbase = (long long)n * args.s_n + (long long)(y * args.out_w + x) * args.s_p;
                if constexpr (EPC > 0) {
                    if (tstore) {
                        epi_stage_bf16_row<EPC>(taddr + a * args.acc_stride + cb_, row_ok,
                                                stg + (uint32_t)(a * args.st_tile_bytes), yy * args.out_w + xx, cb_,
                                                args.st_cw, args.st_chunk_bytes, smem_u32(bs + cb_),
                                                args.bias != nullptr, args.relu != 0);
                        continue;
                    }
                    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out) + rbase + cbase + cb_;
                    if (args.epi_coal)
                        epi_store_bf16_rowseg_coal<EPC>(taddr + a * args.acc_stride + cb_, row_ok, dst,
                                                        smem_u32(bs + cb_), args.bias != nullptr, args.relu != 0,
                                                        stg + (uint32_t)((warp - 4) * coal_warp_bytes<EPC>()), lane);
                    else
                        epi_store_bf16_rowseg<EPC>(taddr + a * args.acc_stride + cb_, row_ok, dst,
                                                   smem_u32(bs + cb_), args.bias != nullptr, args.relu != 0);
                } else if (cb_ < ce_) {
                    epi_store_strided(args, taddr + a * args.acc_stride, row_ok, rbase, col0, cbase, bs, cb_, ce_);
                }
            }
            tc_fence_before();
            if (CG == 2) mbar_arrive_cluster(tempty_leader + (uint32_t)acc * 8u);
            else mbar_arrive(&tempty[acc]);
            if (++acc == nslots) { acc = 0; acc_phase ^= 1; }
            if (tstore) {   // staged tiles -> global: one 4-D tensor store per channel chunk
                fence_proxy_async_smem();
                asm volatile("bar.sync %0, %1;" ::"r"(1 + NEG), "r"(128 * NEG) : "memory");
                if (issuer) {
                    const int cw = args.st_cw > 0 ? (1 << args.st_cw) : EPC;
                    const int nch = args.BN / cw;
                    for (int a = 0; a < macc; a++) {
                        const int tile = tg * tiles_per_unit + (merge ? (int)rank * macc + a : a * CG + (int)rank);
                        if (tile >= args.total_tiles) continue;
                        const int n = tile / args.tiles_per_img;
                        const int y0 = (tile - n * args.tiles_per_img) * args.halo_th;
                        for (int ch = 0; ch < nch; ch++)
                            tma_store_4d(&mapC, stg + (uint32_t)(a * args.st_tile_bytes + ch * args.st_chunk_bytes),
                                         cbase + ch * cw, 0, y0, n);
                    }
                    tma_store_commit();
                }
            }
        }
        if (tstore && issuer) tma_store_wait_all();
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

// ------------------------------------------------------------------ data gradient, column taps in N
// The halo kernel above issues one MMA per filter tap with N = the group's channels: CaffeNet
// conv2's data gradient has 48 per group, 24 per CTA of a pair, so each MMA reads a 4 KB A tile
// for ~24 cycles of tensor work and the pass is bound by shared-memory operand reads (~49% tensor
// pipe).  Here the KW taps of one filter row share an MMA:
//   P[m][(c, j)] = sum_i sum_o A[m + i*wt][o] * Wf[o][c][i][j]   (N = CPG*KW; A shifted by i*wt rows)
//   dX[m][c]     = sum_{j=0..KW-1} P[m + j][(c, j)]               (epilogue)
// (A = dY padded by k-1-p, Wf the flipped filter, S:154 / P:156).  The MMAs are KW times wider and
// the A tile is read KH instead of KH*KW times per 64-channel block.  Accumulator row m + j is TMEM
// lane m + j: the epilogue takes it from lane + j of its warp by a shuffle and, for the last KW-1
// lanes, from the next warp's first lanes through shared memory.  A valid output (x < OW) only
// reads rows of its own padded output row (x + j < wt), so a tile never needs another tile's rows.
// B = the CPG/2 channels x KW taps of this CTA's half, per (filter row i, 64-channel block), stays
// resident in shared memory; each CTA pair serves one group (pair index mod groups).  Row order of
// a B tile (and so the accumulator column of (c, j)) is c*KW + j: the tile is one 4-D TMA box
// (64 o, KW taps, CPG/2 channels) of the flipped, transposed filter WD[G*Cge][taps][Ogp].
__device__ __forceinline__ uint4 jn_pack8(const float (&f)[8]) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; e++) h[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    return u;
}

template <int KH, int KW, int CPG>
__global__ void __launch_bounds__(384, 1)
    tc_halo_jn_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      const TcArgs args) {
    constexpr int CH = 64;
    constexpr int NCOL = KW * CPG;              // MMA N over the pair
    constexpr int B_TILE = NCOL / 2 * 128;      // this CTA's rows of one (i, channel block) tile
    constexpr int CE = CPG / 2;                 // channels per epilogue group
    constexpr int NSUB = CE / 8;                // 8-channel sub-chunks per group
    constexpr int XROW = (KW - 1) * 32 + 16;    // bytes one publishing lane writes per sub-chunk (+ pad)
    constexpr int XWB = (KW - 1) * XROW;        // bytes per warp per sub-chunk
    static_assert(NCOL <= 256 && NCOL % 16 == 0 && (NCOL / 2) % 8 == 0 && CE % 8 == 0, "tile shape");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + HALO_SMEM_ALIGN - 1) &
                                               ~uintptr_t(HALO_SMEM_ALIGN - 1));
    const int cblocks = args.a_cblocks;
    const int a_stages = args.a_stages;
    const int slot = args.halo_slot;
    uint8_t* b_res = smem;                                   // KH * cblocks tiles
    uint8_t* a_ring = b_res + KH * cblocks * B_TILE;
    uint64_t* fullA = reinterpret_cast<uint64_t*>(a_ring + a_stages * slot);
    uint64_t* emptyA = fullA + 4;
    uint64_t* fullB = emptyA + 4;
    uint64_t* tfull = fullB + 1;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    const uint32_t xbase = smem_u32(fullA + 16);             // [2][8 warps][XWB bytes] exchange rows

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
    const int G = args.groups;
    const int g = cid % G, npg = ncl / G;                   // host: ncl is a multiple of G
    const int tgroups = (args.total_tiles + 1) / 2;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
        for (int i = 0; i < a_stages; i++) { mbar_init(&fullA[i], 2); mbar_init(&emptyA[i], 1); }
        mbar_init(fullB, 2);
        for (int i = 0; i < 2; i++) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 128 * 2 * 2); }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_cg2(tmem_holder, 512);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    pdl_wait_and_trigger();

    if (warp == 0 && lane == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (leader) mbar_arrive_expect_tx(fullB, (uint32_t)B_TILE * 2u * (uint32_t)(KH * cblocks));
        else mbar_arrive_cluster(mapa_shared(smem_u32(fullB), 0));
        for (int i = 0; i < KH; i++)
            for (int cb = 0; cb < cblocks; cb++)
                tma_load_4d_cg2(b_res + (i * cblocks + cb) * B_TILE, &mapB, fullB, cb * CH, i * KW,
                                g * args.b_row_g + (int)rank * CE, 0);
        const uint32_t txA = (uint32_t)(args.halo_rows * args.halo_wt * 128);
        int sa = 0;
        uint32_t pa = 0;
        for (int tg = cid / G; tg < tgroups; tg += npg) {
            int tile = tg * 2 + (int)rank;
            if (tile >= args.total_tiles) tile = args.total_tiles - 1;   // rows discarded
            const int n = tile / args.tiles_per_img;
            const int y0 = (tile - n * args.tiles_per_img) * args.halo_th;
            for (int cb = 0; cb < cblocks; cb++) {
                mbar_wait(&emptyA[sa], pa ^ 1);
                if (leader) mbar_arrive_expect_tx(&fullA[sa], txA * 2u);
                else mbar_arrive_cluster(mapa_shared(smem_u32(&fullA[sa]), 0));
                tma_load_4d_cg2(a_ring + sa * slot, &mapA, &fullA[sa], g * args.a_cpg + cb * CH, -args.a_pad_w,
                                y0 - args.a_pad_h, n);
                if (++sa == a_stages) { sa = 0; pa ^= 1; }
            }
        }
    } else if (warp == 1 && leader) {
        // ===================== MMA issuer (leader CTA, whole warp) =====================
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NCOL >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);
        const uint32_t a_base = smem_u32(a_ring), b_base = smem_u32(b_res);
        const uint32_t rowsh = (uint32_t)args.halo_wt * 128u;
        mbar_wait(fullB, 0);
        tc_fence_after();
        int sa = 0, acc = 0, iters = 0;
        uint32_t pa = 0, acc_phase = 0;
        for (int tg = cid / G; tg < tgroups; tg += npg, iters++) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)acc * 256u;
            for (int cb = 0; cb < cblocks; cb++) {
                mbar_wait(&fullA[sa], pa);
                tc_fence_after();
                const uint32_t sa_addr = a_base + (uint32_t)(sa * slot);
                if (elect_one()) {
#pragma unroll
                    for (int i = 0; i < KH; i++) {
                        const uint64_t ad = smem_desc_sw128(sa_addr + (uint32_t)i * rowsh, 16, 1024);
                        const uint64_t bd = smem_desc_sw128(b_base + (uint32_t)((i * cblocks + cb) * B_TILE), 16, 1024);
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            umma_cg2<2>(d, ad + 2 * k, bd + 2 * k, idesc, (cb > 0 || i > 0 || k > 0) ? 1u : 0u);
                    }
                    umma_commit_cg2(&emptyA[sa]);
                }
                __syncwarp();
                if (++sa == a_stages) { sa = 0; pa ^= 1; }
            }
            if (elect_one()) umma_commit_cg2(&tfull[acc]);
            __syncwarp();
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        // the peer's epilogue arrives remotely on our tempty barriers: drain before teardown
        for (int j = iters - 2; j < iters; j++)
            if (j >= 0) mbar_wait(&tempty[j & 1], (uint32_t)((j >> 1) & 1));
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs): 2 groups x 4 warps =====================
        const int q = warp & 3;
        const int eg = (warp - 4) >> 2;
        const int ws = warp - 4;
        const int row = q * 32 + lane;
        const int yy = row / args.halo_wt, xx = row - yy * args.halo_wt;
        const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);
        int acc = 0, xs = 0;
        uint32_t acc_phase = 0;
        for (int tg = cid / G; tg < tgroups; tg += npg) {
            const int tile = tg * 2 + (int)rank;
            const int n = tile / args.tiles_per_img;
            const int y = (tile - n * args.tiles_per_img) * args.halo_th + yy;
            const bool row_ok = tile < args.total_tiles && yy < args.halo_th && y < args.out_h && xx < args.out_w;
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out) + (long long)n * args.s_n +
                                 (long long)(y * args.out_w + xx) * args.s_p + g * args.col_g + eg * CE;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)acc * 256u + (uint32_t)(eg * CE * KW);
#pragma unroll 1
            for (int s = 0; s < NSUB; s++) {
                uint32_t v[8 * KW];
                const uint32_t ta = taddr + (uint32_t)(s * 8 * KW);
#pragma unroll
                for (int c = 0; c + 16 <= 8 * KW; c += 16) tmem_ld16p(ta + c, v + c);
                if constexpr ((8 * KW) % 16 == 8) tmem_ld8p(ta + 8 * KW - 8, v + 8 * KW - 8);
                tmem_wait_ld();
                // publish this warp's first KW-1 lanes for the warp below (rows 32q-KW+1 .. 32q-1 need
                // them): per lane XROW bytes = (j, 8 channels) float rows, 16-byte vector stores; the
                // 16-byte pad per lane puts the lanes of one vector access in distinct banks
                const uint32_t xw = xbase + (uint32_t)((xs * 8 + ws) * XWB);
                if (lane < KW - 1) {
#pragma unroll
                    for (int j = 1; j < KW; j++) {
                        const uint32_t a = xw + (uint32_t)(lane * XROW + (j - 1) * 32);
                        sts_u4(a, v[0 * KW + j], v[1 * KW + j], v[2 * KW + j], v[3 * KW + j]);
                        sts_u4(a + 16, v[4 * KW + j], v[5 * KW + j], v[6 * KW + j], v[7 * KW + j]);
                    }
                }
                float sh[KW - 1][8];   // accumulator row lane + j of this warp
#pragma unroll
                for (int j = 1; j < KW; j++)
#pragma unroll
                    for (int cc = 0; cc < 8; cc++) sh[j - 1][cc] = __shfl_down_sync(0xffffffffu, __uint_as_float(v[cc * KW + j]), j);
                asm volatile("bar.sync %0, 128;" ::"r"(1 + eg) : "memory");
                // rows past this warp's lanes come from the next warp of the group; in the last quadrant
                // they would be rows >= 128, which no valid output reads (x + j < wt)
                if (q < 3 && lane >= 32 - (KW - 1)) {
                    const uint32_t xn = xw + (uint32_t)XWB;
#pragma unroll
                    for (int j = 1; j < KW; j++) {
                        if (lane + j >= 32) {
                            const uint32_t a = xn + (uint32_t)((lane + j - 32) * XROW + (j - 1) * 32);
                            const float4 x0 = lds_f4(a), x1 = lds_f4(a + 16);
                            sh[j - 1][0] = x0.x; sh[j - 1][1] = x0.y; sh[j - 1][2] = x0.z; sh[j - 1][3] = x0.w;
                            sh[j - 1][4] = x1.x; sh[j - 1][5] = x1.y; sh[j - 1][6] = x1.z; sh[j - 1][7] = x1.w;
                        }
                    }
                }
                float o[8];
#pragma unroll
                for (int cc = 0; cc < 8; cc++) {
                    float sum = __uint_as_float(v[cc * KW]);
#pragma unroll
                    for (int j = 1; j < KW; j++) sum += sh[j - 1][cc];
                    o[cc] = sum;
                }
                if (row_ok) *reinterpret_cast<uint4*>(dst + s * 8) = jn_pack8(o);
                xs ^= 1;
            }
            tc_fence_before();
            mbar_arrive_cluster(tempty_leader + (uint32_t)acc * 8u);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_cg2(tmem_base, 512);
    }
}

size_t tc_halo_jn_smem_bytes(const TcArgs& a, int kh, int kw, int cpg) {
    const int xwb = (kw - 1) * ((kw - 1) * 32 + 16);
    return (size_t)kh * a.a_cblocks * (kw * cpg / 2 * 128) + (size_t)a.a_stages * a.halo_slot + 128 /*barriers*/ +
           2 * 8 * xwb + HALO_SMEM_ALIGN;
}

bool tc_halo_jn_compiled(int kh, int kw, int cpg) { return kh == 5 && kw == 5 && cpg == 48; }

cudaError_t tc_halo_jn_launch(const TcLaunch& L, cudaStream_t s) {
    const TcArgs& a = L.args;
    if (!tc_halo_jn_compiled(a.halo_kh, a.a_kw, a.N)) return cudaErrorInvalidValue;
    auto kern = tc_halo_jn_kernel<5, 5, 48>;
    const size_t smem = tc_halo_jn_smem_bytes(a, 5, 5, 48);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_tc(kern, L.grid, 384, smem, s, 2, L.mapA, L.mapB, L.args);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------ weight gradient (halo along K)
// dW[(tap, c)][o] = sum_pixels X[pixel + shift(tap)][c] * dY[pixel][o]: the reduction index is the
// pixel, so a K block is one output tile -- halo_th rows x halo_wt columns (columns >= OW are
// zero-filled in the dY box and contribute nothing).  Its input window (one 64-channel block,
// Cgp == 64) is staged ONCE and serves every tap: the MN-major A operand of tap t is the window
// shifted by shift(t) = i*halo_wt + j rows, and an M=128 tile pairs two taps' 64-channel chunks
// (the descriptor's leading byte offset = the distance between their shifted starts).  A unit
// holds up to MACC such pairs (accumulators, single TMEM buffer) for one o-block, one 64-channel
// block and a split of the pixel tiles; a tile has KSTEPS*16 pixel rows (halo_th whole output rows
// -- for 13x13 maps one whole image, 208 rows).  Partials [unit][BN][128] use the one-pair unit
// index ((split*G + g)*(cblocks*pairs) + cb*pairs + pair)*n_tiles + n_tile; wgrad_reduce's
// cb-major pair mode maps them back.  Rows of the staged tiles beyond the TMA boxes are zeroed
// once and never written.
template <int MACC, int KST>
__global__ void __launch_bounds__(256, 1)
    tc_halo_wgrad_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                         const TcArgs args) {
    // K steps of 16 pixel rows per tile: compile-time when KST > 0 (straight-line issue loop)
    const int ksteps = KST > 0 ? KST : args.halo_ksteps;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + HALO_SMEM_ALIGN - 1) &
                                               ~uintptr_t(HALO_SMEM_ALIGN - 1));
    const int stages = args.stages;
    const int slot = args.halo_slot;                       // A window bytes
    const int bchunk = args.b_stage_bytes / args.b_nchunks; // one 64-channel dY chunk: 128 rows x 128 B
    const int stage_bytes = slot + args.b_stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + stages;
    uint64_t* tfull = empty + stages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 1);
    uint8_t* ones = smem + stages * stage_bytes + 1024;   // 16 rows x 128 B of bf16 1.0

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int taps = args.halo_kh * args.a_kw;
    const int pairs = args.m_tiles_real;
    const int mgroups = args.m_tiles;
    const int cblocks = args.a_cblocks > 0 ? args.a_cblocks : 1;
    const int units = args.groups * args.n_tiles * mgroups * cblocks * args.splits;

    // zero the staging ring once: rows outside the TMA boxes must read as 0 (finite) forever
    {
        uint4* z = reinterpret_cast<uint4*>(smem);
        const int n16 = stages * stage_bytes / 16;
        for (int i = threadIdx.x; i < n16; i += blockDim.x) z[i] = make_uint4(0, 0, 0, 0);
        uint4* o4 = reinterpret_cast<uint4*>(ones);
        for (int i = threadIdx.x; i < 2048 / 16; i += blockDim.x) o4[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
        for (int i = 0; i < stages; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 128);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_holder, args.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    pdl_wait_and_trigger();

    auto decode = [&](int u, int& n_tile, int& mg, int& cb, int& g, int& t0, int& t1) {
        int t = u;
        n_tile = t % args.n_tiles; t /= args.n_tiles;
        mg = t % mgroups; t /= mgroups;
        cb = t % cblocks; t /= cblocks;
        g = t % args.groups;
        const int split = t / args.groups;
        t0 = split * args.kb_per_split;
        t1 = min(args.total_tiles, t0 + args.kb_per_split);
    };

    if (warp == 0 && lane == 0) {
        // ===================== TMA producer =====================
        const uint32_t tx = (uint32_t)(args.halo_rows * args.halo_wt * 128 +
                                       args.b_nchunks * args.halo_th * args.halo_wt * 128);
        int stage = 0;
        uint32_t phase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int n_tile, mg, cb, g, t0, t1;
            decode(u, n_tile, mg, cb, g, t0, t1);
            for (int tile = t0; tile < t1; tile++) {
                const int n = tile / args.tiles_per_img;
                const int y0 = (tile - n * args.tiles_per_img) * args.halo_th;
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_arrive_expect_tx(&full[stage], tx);
                uint8_t* sa = smem + stage * stage_bytes;
                tma_load_4d(sa, &mapA, &full[stage], g * args.a_cpg + cb * 64, -args.a_pad_w, y0 - args.a_pad_h, n);
                for (int c = 0; c < args.b_nchunks; c++)
                    tma_load_4d(sa + slot + c * bchunk, &mapB, &full[stage], g * args.b_col_g + n_tile * args.BN + c * 64,
                                0, y0, n);
                if (++stage == stages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (whole warp, one elected lane issues) =====================
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                               ((uint32_t)(args.BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t base = smem_u32(smem);
        int stage = 0;
        uint32_t phase = 0, acc_phase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int n_tile, mg, cb, g, t0, t1;
            decode(u, n_tile, mg, cb, g, t0, t1);
            const int pa0 = mg * pairs / mgroups, pa1 = (mg + 1) * pairs / mgroups;
            // per accumulator: shifted start (bytes) of its first chunk and the distance to its second
            uint32_t off[MACC], lbo[MACC];
#pragma unroll
            for (int a = 0; a < MACC; a++) {
                const int q0 = 2 * (pa0 + a), q1 = q0 + 1;
                const int s0 = (q0 / args.a_kw) * args.halo_wt + q0 % args.a_kw;
                const int s1 = q1 < taps ? (q1 / args.a_kw) * args.halo_wt + q1 % args.a_kw : s0 + 1;
                off[a] = (uint32_t)s0 * 128u;
                lbo[a] = (uint32_t)(s1 - s0) * 128u;
            }
            mbar_wait(tempty, acc_phase ^ 1);
            tc_fence_after();
            for (int tile = t0; tile < t1; tile++) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t sa = base + stage * stage_bytes;
                const uint64_t bd0 = smem_desc_sw128(sa + slot, (uint32_t)bchunk, 1024);
                // descriptors built by the whole (converged) warp: uniform registers, no per-MMA
                // register->uniform transfer inside the elected lane's issue sequence
                uint64_t ad[MACC];
#pragma unroll
                for (int a = 0; a < MACC; a++) ad[a] = smem_desc_sw128(sa + off[a], lbo[a], 1024);
                const uint32_t first = tile > t0 ? 1u : 0u;
                // the bias accumulator: last pair of channel block 0 with an odd tap count -- its second
                // chunk is the constant ones block, reached by a per-K-step leading byte offset
                const int abias = (args.bias_mma && cb == 0 && pa1 == pairs) ? (pairs - 1 - pa0) : -1;
                const uint32_t ones_addr = smem_u32(ones);
                if (elect_one()) {
#pragma unroll
                    for (int a = 0; a < MACC; a++) {
                        if (a < pa1 - pa0) {
                            const uint32_t dt = tmem_base + a * args.acc_stride;
                            if (a == abias) {
                                for (int k = 0; k < ksteps; k++) {
                                    const uint32_t st0 = sa + off[a] + (uint32_t)k * 2048u;
                                    umma<2>(dt, smem_desc_sw128(st0, ones_addr - st0, 1024), bd0 + (uint64_t)(k * 128),
                                            idesc, (k > 0 || first) ? 1u : 0u);
                                }
                                continue;
                            }
                            umma<2>(dt, ad[a], bd0, idesc, first);
                            if (KST > 0) {
#pragma unroll
                                for (int k = 1; k < (KST > 0 ? KST : 1); k++)
                                    umma<2>(dt, ad[a] + (uint64_t)(k * 128), bd0 + (uint64_t)(k * 128), idesc, 1u);
                            } else {
                                for (int k = 1; k < ksteps; k++)
                                    umma<2>(dt, ad[a] + (uint64_t)(k * 128), bd0 + (uint64_t)(k * 128), idesc, 1u);
                            }
                        }
                    }
                    umma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == stages) { stage = 0; phase ^= 1; }
            }
            if (elect_one()) umma_commit(tfull);
            __syncwarp();
            acc_phase ^= 1;
        }
    } else if (warp >= 4) {
        // ===================== epilogue: FP32 partials =====================
        const int q = warp - 4;
        const int row = q * 32 + lane;
        uint32_t acc_phase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int n_tile, mg, cb, g, t0, t1;
            decode(u, n_tile, mg, cb, g, t0, t1);
            const int split = t0 / args.kb_per_split;
            const int pa0 = mg * pairs / mgroups, pa1 = (mg + 1) * pairs / mgroups;
            mbar_wait(tfull, acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16);
            for (int a = 0; a < pa1 - pa0; a++) {
                const size_t vu = (((size_t)split * args.groups + g) * (cblocks * pairs) + cb * pairs + (pa0 + a)) *
                                      args.n_tiles + n_tile;
                float* dst = args.partial + vu * args.BN * 128 + row;
                for (int c0 = 0; c0 < args.BN; c0 += 32) {
                    const bool two = c0 + 16 < args.BN;
                    uint32_t v0[16], v1[16];
                    tmem_ld16(taddr + a * args.acc_stride + c0, v0);
                    if (two) tmem_ld16(taddr + a * args.acc_stride + c0 + 16, v1);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; j++) dst[(size_t)(c0 + j) * 128] = __uint_as_float(v0[j]);
                    if (two) {
#pragma unroll
                        for (int j = 0; j < 16; j++) dst[(size_t)(c0 + 16 + j) * 128] = __uint_as_float(v1[j]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty);
            acc_phase ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, args.tmem_cols);
    }
}

size_t tc_halo_wgrad_smem_bytes(const TcArgs& a) {
    return (size_t)a.stages * (a.halo_slot + a.b_stage_bytes) + 1024 /*barriers*/ + 2048 /*ones*/ + HALO_SMEM_ALIGN;
}

template <int MACC, int KST>
static cudaError_t halo_wgrad_launch_one(const TcLaunch& L, cudaStream_t s) {
    auto kern = tc_halo_wgrad_kernel<MACC, KST>;
    const size_t smem = tc_halo_wgrad_smem_bytes(L.args);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_tc(kern, L.grid, 256, smem, s, 1, L.mapA, L.mapB, L.args);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

template <int MACC>
static cudaError_t halo_wgrad_dispatch_k(const TcLaunch& L, cudaStream_t s) {
    switch (L.args.halo_ksteps) {
        case 8: return halo_wgrad_launch_one<MACC, 8>(L, s);
        case 11: return halo_wgrad_launch_one<MACC, 11>(L, s);   // conv1 (s2d 57-wide, 3-row tiles)
        case 13: return halo_wgrad_launch_one<MACC, 13>(L, s);   // 13x13 maps, whole image
        case 14: return halo_wgrad_launch_one<MACC, 14>(L, s);   // conv2 (31-wide, 7-row tiles)
        default: return halo_wgrad_launch_one<MACC, 0>(L, s);
    }
}

cudaError_t tc_halo_wgrad_launch(const TcLaunch& L, cudaStream_t s) {
    switch (L.args.macc) {
        case 1: return halo_wgrad_launch_one<1, 0>(L, s);
        case 2: return halo_wgrad_launch_one<2, 0>(L, s);
        case 3: return halo_wgrad_launch_one<3, 0>(L, s);
        case 4: return halo_wgrad_dispatch_k<4>(L, s);
        case 5: return halo_wgrad_dispatch_k<5>(L, s);
        default: return cudaErrorInvalidValue;
    }
}

// Columns per epilogue group of the specialised epilogue, or 0 for the generic one: BF16
// channels-last output, beta 0, no column tail, 16-byte row segments, CTA pairs with two
// accumulators per unit, and a compiled instance for BN/2.
int halo_fast_epc(const TcArgs& a, int cg) {
    const int macc = a.macc > 1 ? a.macc : 1;
    if (!g_halo_fast_epi || cg != 2 || macc != 2 || a.relu_top) return 0;
    if (!(a.out_bf16 && a.s_c == 1 && a.beta == 0.f && a.N % a.BN == 0 && (a.BN / 2) % 8 == 0 && a.s_n % 8 == 0 &&
          a.s_p % 8 == 0 && a.col_g % 8 == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0))
        return 0;
    if (a.epi_groups >= 3)   // three / four epilogue groups: compiled for the 96-column first layer only
        return (a.k_last == 3 && a.a_cblocks == 1 && a.BN == 96 && !a.tma_store) ? 96 / a.epi_groups : 0;
    const int epc = a.BN / 2;
    if (a.k_last == 3 && a.a_cblocks == 1) return (epc == 48 || epc == 64) ? epc : 0;
    return (epc == 24 || epc == 48 || epc == 64) ? epc : 0;
}

template <int CG, int MACC, int KS, int EPC = 0, int BT = 1, int NEG = 2>
static cudaError_t halo_launch_one(const TcLaunch& L, cudaStream_t s) {
    auto kern = tc_halo_kernel<CG, MACC, KS, EPC, BT, NEG>;
    constexpr int threads = 128 + 128 * NEG;
    const size_t smem = tc_halo_smem_bytes(L.args);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_tc(kern, L.grid, threads, smem, s, CG, L.mapA, L.mapB, L.mapC, L.args);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

cudaError_t tc_halo_launch(const TcLaunch& L, cudaStream_t s) {
    if (L.esz != 2) return cudaErrorInvalidValue;
    const int macc = L.args.macc > 1 ? L.args.macc : 1;
    if (macc > 2) return cudaErrorInvalidValue;
    const TcArgs& a = L.args;
    const int epc = halo_fast_epc(a, L.cg);
    if (epc > 0) {
        if (a.k_last == 3 && a.a_cblocks == 1) {
            if (epc == 32 && a.epi_groups == 3) return halo_launch_one<2, 2, 3, 32, 1, 3>(L, s);
            if (epc == 24 && a.epi_groups == 4) return halo_launch_one<2, 2, 3, 24, 1, 4>(L, s);
            if (epc == 48) return halo_launch_one<2, 2, 3, 48>(L, s);
            if (epc == 64) return halo_launch_one<2, 2, 3, 64>(L, s);
        } else {
            if (epc == 24) return a.b_taps == 5 ? halo_launch_one<2, 2, 4, 24, 5>(L, s) : halo_launch_one<2, 2, 4, 24>(L, s);
            if (epc == 48) return halo_launch_one<2, 2, 4, 48>(L, s);
            if (epc == 64) return halo_launch_one<2, 2, 4, 64>(L, s);
        }
    }
    if (L.args.k_last == 3 && L.args.a_cblocks == 1) {
        if (L.cg == 2) return macc == 2 ? halo_launch_one<2, 2, 3>(L, s) : halo_launch_one<2, 1, 3>(L, s);
        return macc == 2 ? halo_launch_one<1, 2, 3>(L, s) : halo_launch_one<1, 1, 3>(L, s);
    }
    if (L.cg == 2) return macc == 2 ? halo_launch_one<2, 2, 4>(L, s) : halo_launch_one<2, 1, 4>(L, s);
    return macc == 2 ? halo_launch_one<1, 2, 4>(L, s) : halo_launch_one<1, 1, 4>(L, s);
}

}  // namespace cb
