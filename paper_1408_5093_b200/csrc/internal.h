// internal.h -- declarations shared by the C-ABI host code and the kernel files.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>
#include "caffe_b200.h"

namespace cb {

// ------------------------------------------------------------------ tensor-core GEMM (tc_gemm.cu)
// D[m, n] = sum_k A[m, k] * B[n, k], A/B staged by TMA in 128-byte-swizzled shared memory,
// tcgen05.mma (M=128, N=BN, K=16 bf16 / 8 tf32) accumulating FP32 in TMEM.
enum AMode { A_TILED_K = 0, A_IM2COL_K = 1, A_IM2COL_MN = 2, A_TILED_MN = 3, A_HALO_K = 4, A_HALO_MN = 5,
             A_HALO_JN = 6 /* data gradient, a filter row's taps in N (tc_halo_jn_kernel) */ };
enum BMode { B_TILED_K = 0, B_TILED_MN = 1 };
enum EpiMode { EPI_STRIDED = 0, EPI_PARTIAL = 1, EPI_SGD = 2 /* fused inner-product update (its own instance) */ };

struct TcArgs {
    int M, N, BN;                       // valid rows, valid cols (per group), N tile
    int m_tiles, n_tiles, groups, splits, units;
    int kblocks, kb_per_split;          // reduction blocks (of 128 bytes of K per row)
    int stages, b_stage_bytes, acc_stride, tmem_cols;
    // A geometry
    int a_P, a_OW;                      // im2col: pixels per image / output width (m -> n, y, x)
    int a_pad_h, a_pad_w, a_kw, a_cblocks, a_cpg;
    int a_nchunks_total;                // A_IM2COL_MN: number of (tap, channel-block) chunks
    int a_row_g;                        // tiled A: row offset per group
    // B geometry
    int b_row_g;                        // B_TILED_K: row offset per group
    int b_col_g;                        // B_TILED_MN: column offset per group
    int b_nchunks;                      // B_TILED_MN: chunks per tile
    // epilogue
    void* out;
    int out_bf16;
    long long s_n, s_c, s_p;            // element strides of (image, column, pixel)
    int P;                              // pixels per image (m -> image, pixel)
    int col_g;                          // output column offset per group
    const float* bias;
    int relu;
    float beta;
    float* partial;                     // EPI_PARTIAL: [unit][BN][128] fp32
    int spin;                           // MMA thread polls (test_wait) instead of try_wait
    // Multi-accumulator units (A_IM2COL_MN + EPI_PARTIAL, CG=1): a unit covers `macc` consecutive
    // 128-row M tiles; each stage holds macc A tiles and ONE B tile, so B is staged once per macc
    // tiles.  m_tiles then counts groups of macc tiles and m_tiles_real the tiles themselves;
    // partials keep the one-tile unit layout (unit = ((split*G+g)*m_tiles_real+mt)*n_tiles+nt).
    int macc;                           // 0/1 = one accumulator per unit
    int m_tiles_real;
    // A_HALO_K (tc_halo.cu, stride-1 convolution): a tile is halo_th output rows x halo_wt columns
    // (halo_wt = output width + kw - 1; columns >= out_w are discarded) of one image.  Its input
    // window -- halo_rows = halo_th + kh - 1 rows x halo_wt columns x 64 channels -- is staged ONCE
    // per channel block by a 4-D tiled TMA load, and every filter tap (i, j) reads it through a
    // descriptor shifted by (i*halo_wt + j) rows of 128 bytes.
    int halo_wt, halo_th, halo_rows, halo_kh, halo_slot;   // halo_slot: smem bytes per tile (1 KB multiple)
    int tiles_per_img, total_tiles, out_h, out_w;
    int halo_ksteps;                    // A_HALO_MN: K steps (16 pixel rows each) per pixel tile
    int bias_mma;                       // A_HALO_MN, odd taps: the last pair's spare chunk is all ones, so
                                        // its accumulator rows 64-127 hold sum_pixels dY (bias gradient)
    int a_stages;                       // halo stages in the A ring
    int b_taps;                         // A_HALO_K: weight tiles (taps) per B stage (1 when resident)
    int b_resident;                     // A_HALO_K: all B tiles (taps x channel blocks) stay in shared
                                        // memory for the whole kernel (one group, one N tile)
    int tma_store;                      // EPI_STRIDED: store tiles with TMA (mapC; row-major output, beta 0)
    int rows_epi;                       // EPI_STRIDED: row-staged coalesced stores (epi_store_rows)
    int k_last;                         // A_HALO_K: 16-channel K steps needed by the last channel block
                                        // (0 = all 4); 3 with a single block selects the KS = 3 kernel
    // A_HALO_K + tma_store: the tile is staged in shared memory as TMA boxes of st_cw channels x
    // out_w pixels x halo_th rows (swizzled by the box row width: 128/64/32 B, or none when the
    // row is an odd number of 16-byte pieces) and written by 4-D tensor stores through mapC
    int st_cw, st_chunk_bytes, st_tile_bytes;
    // A_HALO_K specialised epilogue (EPC > 0, no TMA store): stores coalesced through a per-warp
    // shared-memory transpose (epi_store_bf16_rowseg_coal)
    int epi_coal;
    // A_HALO_K specialised epilogue: epilogue warp groups (2 = default; 3 = conv1's 96 columns as
    // 3 x 32, 512 threads per CTA)
    int epi_groups;
    // EPI_STRIDED data gradient through a ReLU (caffe_conv_backward_data_relu): the result of the
    // pass is kept where relu_top (same element strides as out) is > 0 and zeroed elsewhere,
    // before beta*old is added
    const void* relu_top;
    int relu_top_bf16;
    // A_HALO_K stacked mode (same-size convolutions on small maps, e.g. 3x3/pad 1 on 13x13): the
    // images are laid end to end in one pixel sequence whose rows are stk_wt = W + pad_w wide (one
    // zero column shared by the right pad of a row and the left pad of the next) and whose images
    // are stk_hs = H + pad_h rows tall (one shared zero row); 128-row tiles run over that sequence
    // regardless of image boundaries.  A tile's window is staged as stk_nb one-row TMA boxes placed
    // so that the tile's first pixel lands at shared-memory row stk_off in every CTA.
    int stk, stk_wt, stk_hs, stk_nimg, stk_nb, stk_off;
    // A_HALO_K, macc > 1: the macc tiles of a CTA are consecutive row blocks of one image staged as
    // ONE window of halo_rows = macc*halo_th + kh - 1 rows (accumulator a reads it shifted by
    // a*halo_th*halo_wt rows); halo_slot is then the whole window's stage
    int a_merge;
    // EPI_STRIDED + tma_store, inner-product weight gradient with the SGD update fused in
    // (caffe_ip_backward_weight_sgd): out = the FP32 master weights W (read and rewritten),
    // sgd_v = momentum (same layout), mapC / mapV / mapWb store W, v and the BF16 copy
    int sgd;
    float* sgd_v;
    float sgd_lr, sgd_mom, sgd_decay, sgd_gs;
};

struct TcLaunch {
    CUtensorMap mapA, mapB, mapC;
    CUtensorMap mapV, mapWb;            // fused SGD epilogue: momentum and BF16-weight stores
    TcArgs args;
    int esz;                            // 2 = bf16 (kind::f16), 4 = fp32 (kind::tf32)
    int amode, bmode, epi;
    int cg;                             // 1 = single CTA (M=128), 2 = CTA pair (cta_group::2, M=256)
    int grid;
};

size_t tc_smem_bytes(const TcArgs& a);
// instrumentation (abi.cu): every kernel launch of the library is counted.
void note_launch();
// CAFFE_TUNE_PDL: tensor-core GEMMs launched with programmatic stream serialization (their prologue --
// barrier init, TMEM allocation, cluster sync -- overlaps the tail of the kernel before them; the
// kernels wait on griddepcontrol.wait before touching global memory)
extern int g_pdl;
template <typename K, typename... Args>
cudaError_t launch_tc(K kern, unsigned grid, unsigned threads, size_t smem, cudaStream_t s, int cluster,
                      Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    unsigned na = 0;
    if (cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        na++;
    }
    if (g_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        na++;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
cudaError_t tc_launch(const TcLaunch& L, cudaStream_t s);
cudaError_t tc_halo_launch(const TcLaunch& L, cudaStream_t s);
cudaError_t tc_halo_wgrad_launch(const TcLaunch& L, cudaStream_t s);
size_t tc_halo_wgrad_smem_bytes(const TcArgs& a);
size_t tc_halo_smem_bytes(const TcArgs& a);
// A_HALO_JN (tc_halo.cu): compiled (kh, kw, channels per group) instances and their shared memory
bool tc_halo_jn_compiled(int kh, int kw, int cpg);
size_t tc_halo_jn_smem_bytes(const TcArgs& a, int kh, int kw, int cpg);
cudaError_t tc_halo_jn_launch(const TcLaunch& L, cudaStream_t s);
size_t halo_coal_bytes(const TcArgs& a);
extern int g_halo_coal;   // CAFFE_TUNE_HALO_COALESCE
extern int g_halo_epi_groups;   // CAFFE_TUNE_HALO_EPI_GROUPS
int halo_fast_epc(const TcArgs& a, int cg);
extern int g_halo_tma_store;   // CAFFE_TUNE_HALO_TMA_STORE
int num_sms();

// TMA descriptor encoders (driver entry points resolved at runtime; no -lcuda needed).
// mn_tf32: the tile feeds a TF32 operand in MN-major form (32-byte-atom 128-byte swizzle, see ptx.cuh)
bool encode_tiled_2d(CUtensorMap* m, int esz, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                     uint32_t box_inner, uint32_t box_outer, bool mn_tf32 = false);
// row-major output matrix [rows][cols] (row pitch = ld elements) for TMA stores: box (128 B of
// columns, 32 rows), 128-byte swizzle
bool encode_store_2d(CUtensorMap* m, int esz, const void* base, uint64_t cols, uint64_t rows, uint64_t ld);
// row-major BF16 matrix, box (32 columns = 64 bytes, 32 rows), 64-byte swizzle (fused SGD: BF16 weights)
bool encode_store_2d_bf16_32(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld);
bool encode_tiled_4d(CUtensorMap* m, int esz, const void* base, int C, int W, int H, int N, uint32_t box_c,
                     uint32_t box_w, uint32_t box_h);
// channels-last output [N][H][W][C] (pixel stride s_p, image stride s_n elements) for TMA stores:
// box (box_c channels, box_w, box_h, 1); swizzle 0 / 32 / 64 / 128 bytes
bool encode_store_4d(CUtensorMap* m, int esz, const void* base, int C, int W, int H, int N, long long s_p,
                     long long s_n, uint32_t box_c, uint32_t box_w, uint32_t box_h, int swizzle_bytes);
bool encode_im2col_4d(CUtensorMap* m, int esz, const void* base, int C, int W, int H, int N, int pad_lo_w,
                      int pad_lo_h, int up_w, int up_h, uint32_t channels, uint32_t pixels, bool mn_tf32 = false);

// element strides of a 4-D blob (n, c, h, w) -> n*sn + c*sc + h*sh + w*sw (32-bit: blobs < 2^31)
struct L4 {
    int sn, sc, sh, sw;
};

// ------------------------------------------------------------------ packing kernels (pack.cu)
// Activation -> packed channels-last operand [N][Hp][Wp][Ctot] in bf16 (esz 2) or tf32-rounded
// fp32 (esz 4); group g's channels start at g*cpg.  Space-to-depth for stride s>1: channel
// (dy*sw+dx)*Cg+c of packed pixel (Y,X) of group g is X[n][g*Cg+c][Y*sh+dy-ph][X*sw+dx-pw] (0 outside);
// for s=1 (sh=sw=1, ph=pw=0) it is a plain transpose and TMA supplies the zero padding.
struct PackGeom {
    int N, C, H, W, G, Cg;              // source geometry
    int sh, sw, ph, pw;                 // s2d block (1,1 = plain) and the pad folded into s2d
    int Hp, Wp, cpg, Ctot;              // packed geometry
};
cudaError_t pack_act(const void* src, int src_bf16, L4 ls, int src_nhwc, void* dst, int dst_esz, const PackGeom& g,
                     cudaStream_t s);
// Channels-last int8 image batch -> packed BF16 operand (same layout as pack_act; exact).
cudaError_t pack_act_i8(const void* src, void* dst, const PackGeom& g, cudaStream_t s);
extern int g_i8_rows;   // CAFFE_TUNE_I8_ROWS
extern int g_rows_cb;   // CAFFE_TUNE_ROWS_CB
// Inverse for the s2d data gradient into a blob of either layout, with beta.
cudaError_t unpack_s2d_grad(const float* T, void* dX, int dx_bf16, int xnhwc, float beta, const PackGeom& g,
                            cudaStream_t s);
// Weights (O, Cg, kh, kw) -> forward B operand [G*Og rows][taps'*Cgp] (s2d-aware, zero K padding).
struct WGeom {
    int O, G, Cg, Og, kh, kw, sh, sw;   // original filter geometry (sh,sw = s2d block)
    int khp, kwp, Cgp, Ogp;             // effective (s2d) kernel, K-padded channels
};
cudaError_t repack_w_fwd(const void* w, int w_bf16, void* dst, int dst_esz, const WGeom& g, cudaStream_t s);
// dgrad B operand [G*Cge rows][taps'*Ogp]: row (g, c''), k = (i',j', o), value = fwd-packed W at
// (g*Og+o, kh'-1-i', kw'-1-j', c'')  (flip + transpose); Cge = Cg*sh*sw.
cudaError_t repack_w_dgrad(const void* w, int w_bf16, void* dst, int dst_esz, const WGeom& g, int Cge,
                           cudaStream_t s);
// Deterministic fixed-order reduction of wgrad partials into dW (O, Cg, kh, kw) fp32 with beta.
// cbmajor = 0: M tile = 2 consecutive chunks of q = tap*cblocks + cb (im2col wgrad);
// cbmajor = 1: M tile (pair) = taps (2p, 2p+1) of one channel block, index cb*pairs + p (halo wgrad).
// db (optional, cbmajor only): db = beta*db + sum_splits of row 64 of the last pair of channel block 0
// (the ones chunk of the halo weight gradient).
cudaError_t wgrad_reduce(const float* partial, float* dW, float beta, const WGeom& g, int m_tiles, int n_tiles,
                         int splits, int BN, int chunk, int cblocks, cudaStream_t s, int cbmajor = 0,
                         float* db = nullptr);
// Fixed-order reduction of split-K GEMM partials ([unit][BN][TM] fp32, unit = (s*m_tiles+mt)*n_tiles+nt)
// into a row-major output (ldo) with bias, beta and ReLU; pC > 0 scatters each row's (c,h,w)-ordered
// columns into an NHWC row of pC channels x pHW pixels.
cudaError_t gemm_partial_reduce(const float* part, int splits, int m_tiles, int n_tiles, int BN, int TM, int M, int N,
                                void* out, int out_bf16, long long ldo, const float* bias, int relu, float beta, int pC,
                                int pHW, cudaStream_t s, const void* mref = nullptr, int mref_bf16 = 0);
// Generic 2-D convert/pad: dst[r][c] (ld_dst, esz) = src[r][c] (ld_src, f32|bf16) for c < cols, 0 up to ld_dst.
cudaError_t convert_pad_2d(const void* src, int src_bf16, long long ld_src, void* dst, int dst_esz,
                           long long ld_dst, long long rows, long long cols, cudaStream_t s);
// NHWC blob -> (N, ld) rows in the (c,h,w) flatten order of S:130, and back (fp32 rows, beta).
cudaError_t nhwc_to_rows(const void* src, int src_bf16, void* dst, int dst_esz, int N, int C, int HW, long long ld,
                         cudaStream_t s);
cudaError_t rows_to_nhwc(const float* src, long long ld, void* dst, int dst_bf16, int N, int C, int HW, float beta,
                         cudaStream_t s);

// ------------------------------------------------------------------ CUDA-core kernels (simple.cu)
struct ConvGeom {
    int N, C, H, W, O, kh, kw, sh, sw, ph, pw, G, OH, OW;
};
cudaError_t fp32_conv_fwd(const void* x, int x_bf16, L4 lx, const void* w, int w_bf16, const float* b, void* y,
                          int y_bf16, L4 ly, int ynhwc, int relu, const ConvGeom& g, cudaStream_t s);
// tf32 = 1: operands rounded to TF32 (cvt.rn.tf32.f32, as the tensor-core packs do) before the FP32 FMA
cudaError_t fp32_conv_dgrad(const void* dy, int dy_bf16, L4 ly, const void* w, int w_bf16, void* dx, int dx_bf16,
                            int xnhwc, float beta, const ConvGeom& g, cudaStream_t s, int tf32 = 0);
cudaError_t fp32_conv_wgrad(const void* x, int x_bf16, L4 lx, const void* dy, int dy_bf16, L4 ly, float* dw,
                            float beta, const ConvGeom& g, cudaStream_t s, int tf32 = 0);
int bias_grad_splits(int N, int O, int P);
extern int g_bias_rows;   // CAFFE_TUNE_BIAS_ROWS
extern int g_bias_split_rows;   // CAFFE_TUNE_BIAS_SPLIT_ROWS
cudaError_t bias_grad(const void* dy, int dy_bf16, int nhwc, float* db, float beta, int N, int O, int P, float* part,
                      cudaStream_t s);
cudaError_t im2col_k(const float* x, int n, const ConvGeom& g, float* col, cudaStream_t s);
cudaError_t col2im_k(const float* col, int n, const ConvGeom& g, float* dx, cudaStream_t s);
cudaError_t relu_fwd(const void* x, void* y, int bf16, int count, cudaStream_t s);
cudaError_t relu_bwd(const void* x, const void* dy, void* dx, int x_bf16, int d_bf16, int count, cudaStream_t s);
struct PoolGeom {
    int N, C, H, W, kh, kw, sh, sw, ph, pw, OH, OW;
};
// mask: int32 absolute h*W+w, or (mask_u8) uint8 window-local (h - hs0)*kw + (w - ws0) with the unclipped window start
cudaError_t maxpool_fwd(const void* x, L4 lx, void* y, int ynhwc, void* mask, int mask_u8, int bf16, const PoolGeom& g,
                        cudaStream_t s);
// top (optional): fuse the backward of the ReLU feeding the pool (window gradient passes iff top > 0)
cudaError_t maxpool_bwd(const void* dy, const void* mask, int mask_u8, const void* top, L4 ly, void* dx, int xnhwc, int bf16,
                        const PoolGeom& g, cudaStream_t s);
cudaError_t avepool_fwd(const void* x, L4 lx, void* y, int ynhwc, int bf16, const PoolGeom& g, cudaStream_t s);
cudaError_t avepool_bwd(const void* dy, L4 ly, void* dx, int xnhwc, int bf16, const PoolGeom& g, cudaStream_t s);
cudaError_t lrn_fwd(const void* x, void* y, float* scale, int bf16, int nhwc, int N, int C, int H, int W, int size,
                    float alpha, float beta, float k, cudaStream_t s);
cudaError_t lrn_bwd(const void* x, const void* y, const void* dy, const float* scale, void* dx, int bf16, int nhwc,
                    int N, int C, int H, int W, int size, float alpha, float beta, float k, cudaStream_t s);
// fused CaffeNet pool (3x3/s2, full windows, U8 mask) + LRN, BF16 channels-last (simple.cu)
bool pool_lrn_fusable(const PoolGeom& g, int size);
extern int g_fused_rb;   // CAFFE_TUNE_FUSED_POOL_ROWS
extern int g_pool_lrn_c16;   // CAFFE_TUNE_POOL_LRN_C16
extern int g_lrn_bwd_c16;   // CAFFE_TUNE_LRN_BWD_C16
cudaError_t pool_lrn_fwd(const void* x, void* p, void* mask, void* y, const PoolGeom& g, int size, float alpha,
                         float beta, float k, cudaStream_t s);
cudaError_t lrn_pool_bwd(const void* p, const void* dn, const void* mask, void* dx, int relu, const PoolGeom& g,
                         int size, float alpha, float beta, float k, cudaStream_t s);
cudaError_t softmax_loss_k(const void* scores, int bf16, const int32_t* labels, float* loss, void* diff,
                           int diff_bf16, int N, int K, cudaStream_t s);
extern int g_sgd_blocks_per_sm;
extern int g_sgd_threads;   // CAFFE_TUNE_SGD_THREADS
extern int g_pool_strip_rows;   // CAFFE_TUNE_POOL_STRIP_ROWS
extern int g_wgrad_reduce_sg_min;   // CAFFE_TUNE_WGRAD_REDUCE_SG
extern int g_wgrad_reduce_rows;   // CAFFE_TUNE_WGRAD_REDUCE_ROWS
extern int g_wgrad_reduce_wide;   // CAFFE_TUNE_WGRAD_REDUCE_WIDE
extern int g_halo_fast_epi;   // CAFFE_TUNE_HALO_FAST_EPI
cudaError_t sgd_k(float* w, const float* g, float* v, void* w_bf16, long long count, float lr, float mom,
                  float decay, float gscale, cudaStream_t s);


// ------------------------------------------------------------------ catalogue layers and solver (catalog.cu)
constexpr int ELT_MAX_INPUTS = CAFFE_ELTWISE_MAX_INPUTS;
enum { ELT_PROD = CAFFE_ELTWISE_PROD, ELT_SUM = CAFFE_ELTWISE_SUM, ELT_MAX = CAFFE_ELTWISE_MAX };
enum { LR_FIXED = CAFFE_LR_FIXED, LR_STEP = CAFFE_LR_STEP, LR_INV = CAFFE_LR_INV };
using LrPolicy = caffe_lr_policy;
using SolverDev = caffe_solver_state;
cudaError_t sigmoid_fwd_k(const void* x, void* y, int bf16, long long n, cudaStream_t s);
cudaError_t sigmoid_bwd_k(const void* y, const void* dy, void* dx, int y_bf16, int d_bf16, long long n, cudaStream_t s);
cudaError_t eltwise_fwd_k(int op, int n_in, const void* const* in, const float* coeff, void* y, int bf16, long long n,
                          cudaStream_t s);
cudaError_t eltwise_bwd_k(int op, int n_in, const void* const* in, const float* coeff, const void* dy,
                          void* const* dx, int bf16, long long n, cudaStream_t s);
cudaError_t hinge_loss_k(const void* scores, int bf16, const int32_t* labels, float* loss, void* diff, int diff_bf16,
                         int N, int K, cudaStream_t s);
double lr_policy_host(const LrPolicy& p, long long it);
cudaError_t solver_begin_k(const LrPolicy& p, SolverDev* st, const float* loss, cudaStream_t s);
cudaError_t solver_end_k(SolverDev* st, cudaStream_t s);
cudaError_t sgd_solver_k(float* w, const float* g, float* v, void* w_bf16, long long count, const SolverDev* st,
                         float mom, float decay, float gscale, cudaStream_t s);

}  // namespace cb
