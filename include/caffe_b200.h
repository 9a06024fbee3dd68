/*
 * caffe_b200.h -- C ABI of the B200-native Caffe convolution hot path.
 *
 * The paper (arXiv 1408.5093, /root/reference/PAPER.md = P:n) defines a layer
 * as "a forward pass that takes the inputs and produces the outputs, and a
 * backward pass that takes the gradient with respect to the output, and
 * computes the gradients with respect to the parameters and to the inputs"
 * (Sec. 3.2) over 4-D blobs (num, channels, height, width) (P:141-147,
 * Sec. 3.1).  The layer formulas follow SPEC.md (S:n) lines cited per call;
 * the readings R1..R20 are listed in DESIGN.md.
 *
 * General conventions (apply to every call):
 *  - Pointers inside caffe_blob and the float/int scalars marked "device" are
 *    DEVICE pointers (cudaMalloc / torch allocations on the current device).
 *    Pointers marked "host" are host pointers.  The caller owns every buffer;
 *    the library never allocates device memory and never synchronizes
 *    ("reserves exactly as much memory as needed").
 *  - Blobs are contiguous, NCHW (index ((n*C+c)*H+h)*W+w) or channels-last NHWC
 *    (caffe_layout).  Every call accepts either layout for every activation/diff blob and
 *    the input and output layouts may differ; weights are always (O, C/g, kh, kw) NCHW-order;
 *    pooling masks follow their top's layout.  Blobs hold < 2^31 elements.
 *  - Asynchrony: CAFFE_OK means the work was ENQUEUED on `stream`.  Kernel
 *    launch failures return CAFFE_E_CUDA.  A NULL stream is the legacy
 *    default stream.
 *  - Errors: all validation is host-only and happens before any launch; on
 *    any error nothing is written.  caffe_last_error() returns a thread-local
 *    message naming the offending argument.
 *  - n == 0 is a no-op returning CAFFE_OK; any other zero axis is
 *    CAFFE_E_SHAPE.
 *  - In-place (aliasing input and output) is allowed only where stated
 *    (ReLU); other overlaps return CAFFE_E_ALIAS.
 *  - Determinism: for fixed inputs, configuration and device the outputs are
 *    bitwise reproducible run to run.  No floating-point atomics.
 *  - Math modes: CAFFE_MATH_FP32 = CUDA-core FP32 FMA reference kernels;
 *    CAFFE_MATH_BF16 / CAFFE_MATH_TF32 = sm_100a tcgen05 tensor-core
 *    implicit GEMM with FP32 accumulation in TMEM.  Operands are rounded
 *    (RNE) to bf16 / tf32 before the MMA (reading R12).  TF32 with BF16
 *    storage is CAFFE_E_DTYPE.  Every TF32 pass runs on the tensor cores
 *    (tcgen05.mma kind::tf32), including the weight gradients and the
 *    inner-product data gradient whose operands are MN-major: those are staged
 *    with the 32-byte-atom 128-byte swizzle, the only shared-memory layout the
 *    tensor core takes for MN-major TF32.
 */
#ifndef CAFFE_B200_H_
#define CAFFE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* caffe_stream_t; /* == cudaStream_t */

#define CAFFE_ABI_VERSION 3

typedef enum {
    CAFFE_OK = 0,
    CAFFE_E_INVALID = 1,   /* NULL pointer, bad enum, missing required argument */
    CAFFE_E_SHAPE = 2,     /* inconsistent or zero (non-batch) dimensions */
    CAFFE_E_PARAM = 3,     /* bad layer parameter (kernel > padded input, even LRN size, C%group...) */
    CAFFE_E_DTYPE = 4,     /* unsupported dtype combination */
    CAFFE_E_ALIGN = 5,     /* pointer not 16-byte aligned (tensor-core paths) */
    CAFFE_E_WORKSPACE = 6, /* workspace missing or smaller than caffe_*_workspace_size */
    CAFFE_E_ALIAS = 7,     /* forbidden overlap between input and output buffers */
    CAFFE_E_CUDA = 8,      /* CUDA runtime/driver error (launch failure, no device) */
    CAFFE_E_ARCH = 9       /* device is not sm_100 */
} caffe_status;

typedef enum { CAFFE_F32 = 0, CAFFE_BF16 = 1, CAFFE_I32 = 2, CAFFE_U8 = 3, CAFFE_I8 = 4 } caffe_dtype;
/* CAFFE_I8: signed 8-bit activations -- integer image data (e.g. mean-subtracted pixels in
   [-128, 127], exact in BF16) accepted only as the bottom of caffe_conv_pack_bottom (channels-last,
   BF16 math), which converts it exactly into the packed BF16 operand, and of the prepacked
   caffe_conv_forward / caffe_conv_backward_weight calls that read that operand.  It halves the
   host->device bytes of an input batch. */

typedef enum { CAFFE_MATH_FP32 = 0, CAFFE_MATH_TF32 = 1, CAFFE_MATH_BF16 = 2 } caffe_math;

typedef struct { int32_t n, c, h, w; } caffe_shape4;

/* Memory order of a blob.  The shape is always the logical (num, channels, height, width)
   of P:142 / S:27; the layout only says how it is stored:
     CAFFE_NCHW: index ((n*C+c)*H+h)*W+w   (the paper's blob; default)
     CAFFE_NHWC: index ((n*H+h)*W+w)*C+c   (channels-last: what the tensor-core convolution
                 reads and writes without a transpose; same values, same semantics). */
typedef enum { CAFFE_NCHW = 0, CAFFE_NHWC = 1 } caffe_layout;

typedef struct {
    void* ptr;          /* device pointer, contiguous in `layout` order */
    caffe_shape4 shape;
    caffe_dtype dtype;
    int32_t layout;     /* caffe_layout */
} caffe_blob;

#define CAFFE_FUSE_RELU 1u /* conv/ip forward: apply max(0, .) in the epilogue */
/* conv forward / backward_weight: the workspace already starts with the tensor-core operand of
   `bottom` written by caffe_conv_pack_bottom (same desc, same bottom data, same workspace), so the
   call does not rebuild it.  Ignored by FP32 math and when the operand is read from bottom directly. */
#define CAFFE_BOTTOM_PREPACKED 2u
/* conv forward / backward_data (tensor-core math): the workspace already holds this pass's weight
   operand, written by caffe_conv_pack_weights (same desc, same weight values, same workspace), so
   the call does not repack the filter.  Ignored by FP32 math. */
#define CAFFE_WEIGHTS_PREPACKED 4u

typedef struct {
    int32_t kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w, group;
    caffe_math math;
    uint32_t flags; /* CAFFE_FUSE_RELU | CAFFE_BOTTOM_PREPACKED | CAFFE_WEIGHTS_PREPACKED */
} caffe_conv_desc;

typedef enum { CAFFE_POOL_MAX = 0, CAFFE_POOL_AVE = 1 } caffe_pool_method;

typedef struct {
    int32_t method; /* caffe_pool_method */
    int32_t kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w;
} caffe_pool_desc;

typedef struct {
    int32_t local_size; /* odd, >= 1 */
    float alpha, beta, k;
} caffe_lrn_desc;

typedef enum { CAFFE_PASS_FORWARD = 0, CAFFE_PASS_BACKWARD_DATA = 1, CAFFE_PASS_BACKWARD_WEIGHT = 2 } caffe_pass;

/* ------------------------------------------------------------------ library */
int32_t caffe_abi_version(void);
/* Thread-local text of the last error returned on this thread ("" if none). */
const char* caffe_last_error(void);
/* Checks that a CUDA device of compute capability 10.0 is current. */
caffe_status caffe_device_check(void);

/* Tuning knobs (process-wide; never change results beyond FP32 summation order, which is still
   deterministic for a fixed setting):
   CAFFE_TUNE_CTA_PAIR: 0 = automatic (default), 1 = force single-CTA M=128 tensor-core tiles,
   2 = force CTA-pair M=256 tiles (tcgen05 cta_group::2) where the kernel supports them. */
#define CAFFE_TUNE_CTA_PAIR 1
/* CAFFE_TUNE_MMA_SPIN: 0 (default) = the MMA-issuing thread waits on its stage barrier with the
   suspending try_wait, 1 = it polls (test_wait). */
#define CAFFE_TUNE_MMA_SPIN 2
/* CAFFE_TUNE_WGRAD_MACC: 128-row M tiles per weight-gradient work unit (top_diff staged once for
   all of them); 0 = automatic (default), 1..4 forced. */
#define CAFFE_TUNE_WGRAD_MACC 3
/* CAFFE_TUNE_HALO: stride-1 forward / data-gradient tensor-core tiles that stage each input window
   once for all filter taps (halo tiles); 0 = automatic (default), 1 = off (per-tap im2col tiles),
   2 = wherever the geometry allows. */
#define CAFFE_TUNE_HALO 4
/* CAFFE_TUNE_TMA_STORE: 1 (default) = tensor-core epilogues of row-major / channels-last outputs
   (beta 0) stage 32-row tiles in shared memory and write them with TMA tensor stores; 0 = direct
   per-thread vector stores.  Bit-identical results. */
#define CAFFE_TUNE_TMA_STORE 5
/* CAFFE_TUNE_ROWS_EPILOGUE: 1 = channels-last BF16 tensor-core outputs (beta 0, <= 128 columns per
   tile) are staged per warp in shared memory and written back in memory order (contiguous 512-byte
   stores when a tile holds whole pixels); 0 (default) = each thread stores its own row.
   Bit-identical results. */
#define CAFFE_TUNE_ROWS_EPILOGUE 6
/* CAFFE_TUNE_SGD_BLOCKS_PER_SM: grid of caffe_sgd_update in 256-thread blocks per SM (0 = default 4).
   1 leaves registers and thread slots for kernels running concurrently on other streams (an update
   overlapped with the backward pass).  Read at launch time. */
#define CAFFE_TUNE_SGD_BLOCKS_PER_SM 7
/* CAFFE_TUNE_POOL_STRIP_ROWS: block rows per thread in the channels-last 3x3/s2 max-pool backward
   (0 = auto).  Results are identical for every value. */
#define CAFFE_TUNE_POOL_STRIP_ROWS 8
/* CAFFE_TUNE_WGRAD_REDUCE_SG: weight-gradient split reductions with at least this many splits use
   several threads per output (fixed-order tree; 0 = default 24).  Deterministic for every value;
   values differ only in the FP32 summation order. */
#define CAFFE_TUNE_WGRAD_REDUCE_SG 9
/* CAFFE_TUNE_HALO_KTRIM: halo-tiled forward / data gradient skip the K steps of the padding
   channels of the last 64-channel block (1 = default, 0 = multiply the zero padding). */
#define CAFFE_TUNE_HALO_KTRIM 10
/* CAFFE_TUNE_HALO_FAST_EPI: 1 (default) = halo-tiled forward / data-gradient kernels with BF16
   channels-last outputs (beta 0, no column tail) use the specialised row-segment epilogue (all TMEM
   loads before one wait, shared-memory bias vectors, 16-byte stores); 0 = the generic epilogue.
   Bit-identical results. */
#define CAFFE_TUNE_HALO_FAST_EPI 11
/* CAFFE_TUNE_HALO_TMA_STORE: 1 = the specialised halo epilogue stages each tile in shared memory and
   writes it with 4-D TMA tensor stores; 0 (default) = per-thread 16-byte global stores (measured:
   equal for conv1, faster for conv2 whose B ring keeps more stages).  Bit-identical results. */
#define CAFFE_TUNE_HALO_TMA_STORE 12
/* CAFFE_TUNE_WGRAD_REDUCE_ROWS: 1 = the split reduction of the halo weight gradients of
   plain filters (fewer splits than CAFFE_TUNE_WGRAD_REDUCE_SG) runs one block per (filter row,
   64-channel block) with a shared-memory gather and contiguous dW stores; 0 (default) = one thread
   per weight (measured slightly faster in the step).  Bit-identical results (same summation order). */
#define CAFFE_TUNE_WGRAD_REDUCE_ROWS 13
/* CAFFE_TUNE_HALO_STACKED: stacked halo tiles for same-size stride-1 convolutions (odd kernel, centred
   padding) on maps too small for whole-row halo tiles (CaffeNet conv3-5 forward and data
   gradient): images laid end to end as one pixel sequence with shared zero rows/columns, one
   staged window per 128-pixel tile serving every tap.  0 = off (per-tap im2col tiles), 1 (default)
   = where whole-row halo tiles do not apply and N tiles are <= 128 columns (CaffeNet conv5
   forward), 2 = wherever the geometry allows, 3 = as 2 with two accumulators per CTA for N tiles of
   up to 256 columns (single-buffered TMEM), 4 = as 2 with wider N split into tiles of <= 128
   columns (two double-buffered accumulators). */
#define CAFFE_TUNE_HALO_STACKED 14
/* CAFFE_TUNE_SGD_THREADS: threads per block of caffe_sgd_update (0 = default 256; 64, 128): with
   CAFFE_TUNE_SGD_BLOCKS_PER_SM it sets how much of an SM an update running beside the backward
   takes.  Results are identical. */
#define CAFFE_TUNE_SGD_THREADS 15
/* CAFFE_TUNE_MAX_CTAS: caps the persistent tensor-core grids at this many CTAs (0 = default, one
   CTA or CTA pair per SM).  Work units, split-K boundaries and reduction orders do not depend on
   it, so results are bit-identical for every value; a small cap makes each CTA loop over many
   units (accumulator double-buffer and barrier phases carried across units), which is how the
   parity tests exercise the batch-256 schedule at small sizes. */
#define CAFFE_TUNE_MAX_CTAS 16
/* CAFFE_TUNE_FUSED_POOL_ROWS: 2x2-block rows per CTA of caffe_lrn_pool_backward (0 = automatic).
   Results are identical for every value. */
#define CAFFE_TUNE_FUSED_POOL_ROWS 17
/* CAFFE_TUNE_HALO_COALESCE: 1 (default) = the specialised halo epilogue transposes each warp's rows
   through shared memory so its global stores are coalesced (conv1's 148.7 MB output); 0 = each
   thread stores its own row.  Bit-identical results. */
#define CAFFE_TUNE_HALO_COALESCE 18
/* CAFFE_TUNE_WGRAD_REDUCE_WIDE: 1 = weight-gradient split reductions with >= 64 / >= 96 splits use
   16 / 32 threads per output (a few partials each); 0 (default, measured faster) = at most 8.
   Deterministic for either value; the two differ only in the FP32 summation order. */
#define CAFFE_TUNE_WGRAD_REDUCE_WIDE 19
/* CAFFE_TUNE_HALO_BTAPS: filter taps' weight tiles per B pipeline stage of the halo-tiled forward /
   data gradient: 0 (default) = 5 where compiled (the 24-column-per-CTA data gradient of 5x5
   filters, CaffeNet conv2) and >= 4 stages fit, else 1; 1 = always one.  Identical results. */
#define CAFFE_TUNE_HALO_BTAPS 20
/* CAFFE_TUNE_HALO_EPI_GROUPS: epilogue warp groups of the halo-tiled forward with 96 output columns
   and one 48-channel block (the space-to-depth first layer): 0 (default) = 3, 2 = two groups of 48
   columns (384 threads), 3 = three groups of 32 (512 threads; conv1 forward 78.4 -> 71.8 us at batch
   256), 4 = four groups of 24 (640 threads).  Identical results. */
#define CAFFE_TUNE_HALO_EPI_GROUPS 21
/* CAFFE_TUNE_HALO_JN: 1 (default) = stride-1 data gradients of compiled shapes (5x5 filters, 48
   channels per group: CaffeNet conv2) run the kernel that puts the kw taps of a filter row in the
   MMA's N (kw x 48 = 240 columns per MMA instead of 48) and sums the taps' shifted accumulator rows
   in the epilogue; 0 = one MMA per tap.  Same result up to FP32 summation order. */
#define CAFFE_TUNE_HALO_JN 22
/* CAFFE_TUNE_WGRAD_BN: output-channel (N) tile of the halo-tiled weight gradients: 0 (default) =
   automatic (several channel blocks: <= 96 columns, five accumulators per unit), 1 = the widest of
   192/128/96/64 dividing the outputs (faster alone, slower in the three-stream training step),
   2 = <= 96 columns but 128 instead of 64 (measured no faster in the step), else a multiple of 16
   up to 256.  Same result up to FP32 summation order. */
#define CAFFE_TUNE_WGRAD_BN 23
/* CAFFE_TUNE_HALO_MERGE: 1 = halo-tiled forward / data-gradient CTAs with two accumulators take two
   consecutive row blocks of one image and stage one shared input window for both, three stages deep
   (where an image has an even number of tiles, e.g. the first layer); 0 (default) = one window per
   tile (measured as fast).  Identical results. */
#define CAFFE_TUNE_HALO_MERGE 24
/* CAFFE_TUNE_IP_MAX_SPLITS: cap on the split-K factor of the inner-product forward / data gradient
   (0 = none: splits fill the CTA pairs).  Same result up to FP32 summation order. */
#define CAFFE_TUNE_IP_MAX_SPLITS 25
/* CAFFE_TUNE_I8_ROWS: 1 (default) = the int8 image pack of a 4x4 space-to-depth of 3 channels (the
   CaffeNet first layer) runs one thread per packed pixel (four 12-byte segments in flight, six
   16-byte stores); 0 = one thread per 12-byte source segment.  Identical results. */
#define CAFFE_TUNE_I8_ROWS 26
/* CAFFE_TUNE_ROWS_CB: 1 (default) = a BF16 channels-last inner-product input is staged as (c,h,w)
   rows by one block per (64-channel block, image) with paired 4-byte stores; 0 = one block per image
   (scalar stores).  Identical results. */
#define CAFFE_TUNE_ROWS_CB 27
/* CAFFE_TUNE_BIAS_ROWS: 1 = an inner product's bias gradient (<= 8192 rows) in one pass (8 row
   groups per column block, fixed order); 0 (default) = split partials + a final pass (the one-pass
   form measured slower in the training step).  Deterministic either way; the FP32 summation order
   differs. */
#define CAFFE_TUNE_BIAS_ROWS 28
/* CAFFE_TUNE_BIAS_SPLIT_ROWS: rows (pixels x images) per split of the two-pass bias gradient, 8 ..
   1024 (default 64).  Deterministic; the FP32 summation order follows the split. */
#define CAFFE_TUNE_BIAS_SPLIT_ROWS 29
/* CAFFE_TUNE_PDL: 1 = the tensor-core GEMMs are launched with programmatic stream serialization, so
   their prologue (barrier init, TMEM allocation, cluster sync) overlaps the end of the kernel before
   them on the stream; they wait for it (griddepcontrol.wait) before touching global memory.
   0 (default) = ordinary stream order.  Identical results. */
#define CAFFE_TUNE_PDL 30
/* CAFFE_TUNE_IP_FWD_SMALL_BN: N tile (64 or 128, default 128) of inner-product forwards with <= 1024
   outputs (fc8: fewer split-K partials to reduce); 0 = the general rule.  Same result up to FP32
   summation order. */
#define CAFFE_TUNE_IP_FWD_SMALL_BN 31
/* CAFFE_TUNE_POOL_LRN_C16: 1 (default) = caffe_pool_lrn_forward with C % 16 == 0 where C/8 does not
   divide 32 (CaffeNet's 96-channel pool1/norm1) and an LRN window of <= 5 runs 16 channels per lane;
   0 = 8 channels per lane.  Identical results. */
#define CAFFE_TUNE_POOL_LRN_C16 32
/* CAFFE_TUNE_LRN_BWD_C16: 1 (default) = the BF16 channels-last LRN backward with C % 16 == 0 runs 16
   channels per lane (own channels loaded once, neighbours by shuffle); 0 = 8 channels per thread
   with the neighbouring vectors loaded.  Identical results. */
#define CAFFE_TUNE_LRN_BWD_C16 33
caffe_status caffe_set_tuning(int32_t key, int32_t value);

/* ------------------------------------------------------------------ instrumentation
   (for benchmarks; never changes results)
   caffe_launch_count: cumulative number of kernels this library launched in the process.
   caffe_profiler_enable(on): on != 0 clears the record list and starts recording a CUDA event
     pair on the call's stream around every tcgen05 GEMM launch, tagged with the call's
     algorithmic FLOPs (2*MACs of the layer pass) and kind (0 = convolution, 1 = inner product);
     on == 0 stops recording.
   caffe_profiler_read(kind, ...): synchronises the recorded events and returns the summed
     duration (ms), summed algorithmic FLOPs and launch count of the records of `kind`
     (-1 = all).  Host pointers. */
int64_t caffe_launch_count(void);
caffe_status caffe_profiler_enable(int32_t on);
caffe_status caffe_profiler_read(int32_t kind, double* ms /* host */, double* flops /* host */,
                                 int64_t* launches /* host */);

/* ------------------------------------------------------------------ convolution
 * Convolution with groups, stride and zero padding (S:145 + reading R3):
 *   top[n,o,y,x] = bias[o] + sum_{c'<C/g,i<kh,j<kw} W[o,c',i,j] *
 *                  bottom[n, (o/(O/g))*(C/g)+c', y*sh-ph+i, x*sw-pw+j]
 * Output size floor((H+2p-k)/s)+1.  Weight blob shape (O, C/g, kh, kw).
 */

/* top shape (host out) for a bottom shape and num_output.  E_PARAM if the kernel
   exceeds the padded input or C % group != 0 or num_output % group != 0. */
caffe_status caffe_conv_output_shape(const caffe_conv_desc* desc, caffe_shape4 bottom, int32_t num_output,
                                     caffe_shape4* top /* host */);

/* Bytes of device workspace the given pass needs (host out).  0 for CAFFE_MATH_FP32
   forward/backward-data.  `weight` is the weight blob shape. */
caffe_status caffe_conv_workspace_size(const caffe_conv_desc* desc, caffe_shape4 bottom, caffe_shape4 weight,
                                       int32_t pass /* caffe_pass */, size_t* bytes /* host */);

/* Builds the tensor-core operand of `bottom` (channels-last, groups padded, space-to-depth for
   strided convs) at the start of `workspace` -- the work caffe_conv_forward and
   caffe_conv_backward_weight repeat for every call -- so both can then run with
   CAFFE_BOTTOM_PREPACKED on that workspace (the first layer's image batch is packed once per
   step instead of twice).  `weight` supplies the filter geometry only.  Workspace: at least the
   larger of the forward and backward-weight sizes.  No-op (CAFFE_OK) for FP32 math or when the
   operand is read from bottom directly. */
caffe_status caffe_conv_pack_bottom(const caffe_conv_desc* desc, const caffe_blob* bottom, const caffe_blob* weight,
                                    void* workspace, size_t workspace_bytes, caffe_stream_t stream);

/* Builds the tensor-core weight operand of one pass -- pass CAFFE_PASS_FORWARD: (O, C/g, kh, kw)
   repacked K-major per tap and channel block; CAFFE_PASS_BACKWARD_DATA: flipped and transposed --
   at its place in `workspace` (the place caffe_conv_forward / caffe_conv_backward_data use), so
   calls with CAFFE_WEIGHTS_PREPACKED on that workspace skip the repack.  The caller repacks after
   every change of the weights (the training step does it right after each layer's update, off the
   critical path).  `bottom` gives the input geometry.  Workspace: the pass's size.  No-op for FP32
   math.  Errors: as the pass itself (E_SHAPE, E_PARAM, E_WORKSPACE, E_ALIGN, E_INVALID for another
   pass). */
caffe_status caffe_conv_pack_weights(const caffe_conv_desc* desc, caffe_shape4 bottom, const caffe_blob* weight,
                                     int32_t pass /* caffe_pass */, void* workspace, size_t workspace_bytes,
                                     caffe_stream_t stream);

/* Forward.  bottom F32|BF16, weight F32|BF16, bias F32 (nullable), top
   F32|BF16 (overwritten).  Fused ReLU with CAFFE_FUSE_RELU. */
caffe_status caffe_conv_forward(const caffe_conv_desc* desc, const caffe_blob* bottom, const caffe_blob* weight,
                                const caffe_blob* bias, caffe_blob* top, void* workspace, size_t workspace_bytes,
                                caffe_stream_t stream);

/* Data gradient: bottom_diff = beta*bottom_diff + conv^T(top_diff) (R4:
   beta = 0 overwrites, Caffe default for data). */
caffe_status caffe_conv_backward_data(const caffe_conv_desc* desc, const caffe_blob* top_diff,
                                      const caffe_blob* weight, caffe_blob* bottom_diff, float beta,
                                      void* workspace, size_t workspace_bytes, caffe_stream_t stream);

/* Data gradient through the ReLU that produced this layer's bottom (S:151-159 with the ReLU
   backward of S:205-213 folded in; the net's in-place ReLU keeps only its output, whose sign is
   the sign of its input):
     bottom_diff = [relu_top > 0] * conv^T(top_diff)        (overwritten; beta is 0)
   relu_top: the ReLU output (= this layer's bottom), F32|BF16, same shape and layout as
   bottom_diff, must not overlap it.  Same workspace as caffe_conv_backward_data.  The mask is
   applied in the tensor-core epilogue where it can (channels-last BF16 im2col / halo tiles),
   else by an in-place ReLU-backward pass after the convolution.  Errors: as
   caffe_conv_backward_data, plus E_SHAPE (relu_top shape), E_INVALID (layouts differ), E_ALIAS. */
caffe_status caffe_conv_backward_data_relu(const caffe_conv_desc* desc, const caffe_blob* top_diff,
                                           const caffe_blob* weight, const caffe_blob* relu_top,
                                           caffe_blob* bottom_diff, void* workspace, size_t workspace_bytes,
                                           caffe_stream_t stream);

/* Weight/bias gradient (accumulate S:154 via beta, R4):
     weight_diff[o,c',i,j] = beta*weight_diff + sum_{n,y,x} top_diff[n,o,y,x]*bottom[n,g(o)C/g+c',y*sh-ph+i,x*sw-pw+j]
     bias_diff[o]          = beta*bias_diff   + sum_{n,y,x} top_diff[n,o,y,x]
   weight_diff and bias_diff are F32; bias_diff nullable.  Deterministic split
   reduction (no atomics). */
caffe_status caffe_conv_backward_weight(const caffe_conv_desc* desc, const caffe_blob* bottom,
                                        const caffe_blob* top_diff, caffe_blob* weight_diff, caffe_blob* bias_diff,
                                        float beta, void* workspace, size_t workspace_bytes, caffe_stream_t stream);

/* ------------------------------------------------------------------ ReLU
   forward: top = bottom > 0 ? bottom : +0 (R10); top may equal bottom (in place).
   backward: bottom_diff = top_diff where x > 0 else 0, x = the forward input or output
   (same sign test); bottom_diff may equal top_diff. */
caffe_status caffe_relu_forward(const caffe_blob* bottom, caffe_blob* top, caffe_stream_t stream);
caffe_status caffe_relu_backward(const caffe_blob* bottom_or_top, const caffe_blob* top_diff, caffe_blob* bottom_diff,
                                 caffe_stream_t stream);

/* ------------------------------------------------------------------ pooling
   Output size: ceil((H+2p-k)/s)+1, minus 1 if (OH-1)*s >= H+p (reading R5).
   MAX: strict '>' row-major scan seeded by the first in-image element; mask =
   int32 h*W+w in the (n,c) plane (R7), mask nullable in forward.  A CAFFE_U8 mask blob stores
   the same argmax as the window-local index (h - (py*sh - ph))*kw + (w - (px*sw - pw)) (requires
   kh*kw <= 255): a quarter of the mask bytes for the backward pass to read; same results.
   AVE: divisor (min(hs+k,H+p)-hs)*(min(ws+k,W+p)-ws) (R6).
   backward overwrites bottom_diff; MAX sums top_diff in ascending (py,px) order
   in FP32 (R8, bit-exact); MAX backward without mask is CAFFE_E_INVALID. */
caffe_status caffe_pool_output_shape(const caffe_pool_desc* desc, caffe_shape4 bottom, caffe_shape4* top /* host */);
caffe_status caffe_pool_forward(const caffe_pool_desc* desc, const caffe_blob* bottom, caffe_blob* top,
                                caffe_blob* mask, caffe_stream_t stream);
caffe_status caffe_pool_backward(const caffe_pool_desc* desc, const caffe_blob* top_diff, const caffe_blob* mask,
                                 caffe_blob* bottom_diff, caffe_stream_t stream);
/* MAX pool backward fused with the backward of the ReLU that produced the pool's bottom
   (conv -> ReLU -> MAX pool, S:196-213 then S:160-177):
   bottom_diff = relu_backward(bottom, pool_backward(top_diff)).  Since the window max `top`
   equals the ReLU output at its argmax, a window passes its gradient iff top > 0 -- the same
   result, bit for bit, as caffe_pool_backward followed by caffe_relu_backward.  `top` is the
   pool forward output (shape, dtype and layout of top_diff).  AVE pooling is CAFFE_E_INVALID. */
caffe_status caffe_pool_relu_backward(const caffe_pool_desc* desc, const caffe_blob* top, const caffe_blob* top_diff,
                                      const caffe_blob* mask, caffe_blob* bottom_diff, caffe_stream_t stream);

/* ------------------------------------------------------------------ LRN (R9)
   S = k + alpha/n * sum_{c' in [c-r, c+r] clipped} x^2, r=(n-1)/2;  top = bottom * S^-beta.
   scale (F32, nullable) receives S.  Backward is the exact derivative:
   bottom_diff = top_diff*S^-beta - (2 alpha beta/n) * x * sum_{c' in win(c)} top_diff*top/S,
   where top/S is evaluated as x*S^-beta/S in FP32 from the bottom (the top blob is validated but
   not read: a BF16-stored top would carry its rounding into that term).
   Even local_size is CAFFE_E_PARAM. */
caffe_status caffe_lrn_forward(const caffe_lrn_desc* desc, const caffe_blob* bottom, caffe_blob* top,
                               caffe_blob* scale, caffe_stream_t stream);
caffe_status caffe_lrn_backward(const caffe_lrn_desc* desc, const caffe_blob* bottom, const caffe_blob* top,
                                const caffe_blob* top_diff, const caffe_blob* scale, caffe_blob* bottom_diff,
                                caffe_stream_t stream);

/* ------------------------------------------------------------------ inner product
   bottom (N,C,H,W) is flattened to (N, K=C*H*W); weight (O,K,1,1); bias (O) F32
   nullable; top (N,O,1,1).  forward top = bottom * W^T + b, CAFFE_FUSE_RELU
   honoured via `flags`; backward_data bottom_diff = beta*bottom_diff + top_diff*W;
   backward_weight weight_diff = beta*weight_diff + top_diff^T*bottom,
   bias_diff = beta*bias_diff + sum_n top_diff. */
caffe_status caffe_ip_workspace_size(caffe_math math, caffe_shape4 bottom, int32_t num_output, int32_t pass,
                                     size_t* bytes /* host */);
caffe_status caffe_ip_forward(caffe_math math, uint32_t flags, const caffe_blob* bottom, const caffe_blob* weight,
                              const caffe_blob* bias, caffe_blob* top, void* workspace, size_t workspace_bytes,
                              caffe_stream_t stream);
caffe_status caffe_ip_backward_data(caffe_math math, const caffe_blob* top_diff, const caffe_blob* weight,
                                    caffe_blob* bottom_diff, float beta, void* workspace, size_t workspace_bytes,
                                    caffe_stream_t stream);
/* Data gradient through the ReLU that produced this layer's bottom (S:187-195 with S:205-213 folded
   in): bottom_diff = [relu_top > 0] * (top_diff . W) (overwritten).  relu_top: the ReLU output
   (= this layer's bottom), F32|BF16, same shape and layout as bottom_diff, no overlap.  The mask is
   applied in the split-K reduce or the tensor-core epilogue where it can, else by an in-place
   ReLU-backward pass.  Errors: as caffe_ip_backward_data, plus E_SHAPE, E_INVALID, E_ALIAS. */
caffe_status caffe_ip_backward_data_relu(caffe_math math, const caffe_blob* top_diff, const caffe_blob* weight,
                                         const caffe_blob* relu_top, caffe_blob* bottom_diff, void* workspace,
                                         size_t workspace_bytes, caffe_stream_t stream);
caffe_status caffe_ip_backward_weight(caffe_math math, const caffe_blob* bottom, const caffe_blob* top_diff,
                                      caffe_blob* weight_diff, caffe_blob* bias_diff, float beta, void* workspace,
                                      size_t workspace_bytes, caffe_stream_t stream);

/* Inner-product weight gradient with the SGD update fused in (S:187-195 then S:520-528; one GPU,
   where nothing needs the gradient itself): for every weight,
     g' = dW*grad_scale + decay*W;  v = momentum*v - lr*g';  W = W + v;  weight_bf16 = RNE(W)
   with dW = top_diff^T . bottom computed by the tensor cores and consumed in the epilogue (never
   stored; bit-identical to caffe_ip_backward_weight followed by caffe_sgd_update).  bias_diff
   (nullable, F32, overwritten) receives the bias gradient; the bias update stays with
   caffe_sgd_update.  weight/momentum F32 and weight_bf16 BF16, all (O, K) row-major, K % 32 == 0,
   16-byte aligned, mutually non-overlapping.  BF16 tensor-core math only.  Errors: E_SHAPE, E_DTYPE,
   E_INVALID (layout), E_ALIGN, E_ALIAS, E_WORKSPACE (size as caffe_ip_workspace_size(BF16, ...,
   CAFFE_PASS_BACKWARD_WEIGHT)). */
caffe_status caffe_ip_backward_weight_sgd(const caffe_blob* bottom, const caffe_blob* top_diff, caffe_blob* weight,
                                          caffe_blob* momentum, caffe_blob* weight_bf16, caffe_blob* bias_diff,
                                          float lr, float momentum_coef, float decay, float grad_scale,
                                          void* workspace, size_t workspace_bytes, caffe_stream_t stream);

/* Layout change (S:130's (c,h,w) order): dst (NCHW, BF16) = src (channels-last, F32|BF16), same
   logical shape, RNE when narrowing: plain (N, C*H*W) inner-product rows from a channels-last map.
   Errors: E_SHAPE, E_INVALID (layouts), E_ALIAS, E_DTYPE (dst not BF16). */
caffe_status caffe_blob_to_nchw(const caffe_blob* src, caffe_blob* dst, caffe_stream_t stream);

/* ------------------------------------------------------------------ im2col / col2im (test entry points)
   S:297 / S:806 lowering of image n: col[(c*kh+i)*kw+j][y*OW+x] = bottom[n,c,y*sh-ph+i,x*sw-pw+j]
   (0 outside), col is an F32 blob of shape (1,1,C*kh*kw,OH*OW).  col2im is its
   adjoint, written as a gather summing in ascending (y, x) order in FP32 into image n
   of bottom_diff (overwritten).  Bit-exact vs the oracle.  group/math ignored. */
caffe_status caffe_im2col(const caffe_conv_desc* desc, const caffe_blob* bottom, int32_t n, caffe_blob* col,
                          caffe_stream_t stream);
caffe_status caffe_col2im(const caffe_conv_desc* desc, const caffe_blob* col, int32_t n, caffe_blob* bottom_diff,
                          caffe_stream_t stream);

/* ------------------------------------------------------------------ glue for the training step
   Softmax with loss: loss (device F32 scalar) = -(1/N) sum_n log softmax(s_n)[l_n];
   score_diff = (softmax - onehot)/N (nullable).  labels: device int32[N] in [0,K).  The labels live
   on the device, so their range cannot be checked before the (asynchronous) launch: a label
   outside [0,K) ("label out of range") is never used as an index; it makes the loss NaN and
   that row of score_diff NaN, which the caller sees on its next read of the loss. */
caffe_status caffe_softmax_loss(const caffe_blob* scores, const int32_t* labels /* device */,
                                float* loss /* device */, caffe_blob* score_diff, caffe_stream_t stream);

/* SGD with momentum and weight decay (reading R18):
   g' = g*grad_scale + decay*w;  v = momentum*v - lr*g';  w = w + v.
   All device F32 of `count` elements; w_bf16 (device, nullable) receives RNE(w) for
   the next step's BF16 operands. */
caffe_status caffe_sgd_update(float* w, const float* g, float* v, void* w_bf16, int64_t count, float lr,
                              float momentum, float decay, float grad_scale, caffe_stream_t stream);

/* ------------------------------------------------------------------ fused pool + LRN
   CaffeNet's "pool -> LRN" blocks (P:158 pooling + local response normalization; S:160-177,
   S:214-231) in one pass each, for BF16 channels-last blobs, MAX 3x3/stride-2 unpadded windows that
   lie inside the map, C % 8 == 0, local_size <= 9 and a U8 window-local mask (anything else:
   CAFFE_E_INVALID / CAFFE_E_DTYPE -- use the separate calls).  Results are bit-identical to the
   separate calls; only the intermediate blob's trip through memory is gone.
   caffe_pool_lrn_forward: pool_top = maxpool(bottom) (+ mask), top = lrn(pool_top).
   caffe_lrn_pool_backward: bottom_diff (pool input diff, overwritten) = maxpool_backward(
     lrn_backward(pool_top, top_diff), mask), with relu != 0 gated as caffe_pool_relu_backward (the
     ReLU that feeds the pool: a window passes its gradient only when pool_top > 0).  pool_top is the
     LRN's bottom, so the LRN backward needs no other blob. */
caffe_status caffe_pool_lrn_forward(const caffe_pool_desc* pool, const caffe_lrn_desc* lrn, const caffe_blob* bottom,
                                    caffe_blob* pool_top, caffe_blob* mask, caffe_blob* top, caffe_stream_t stream);
caffe_status caffe_lrn_pool_backward(const caffe_pool_desc* pool, const caffe_lrn_desc* lrn, const caffe_blob* pool_top,
                                     const caffe_blob* top_diff, const caffe_blob* mask, int32_t relu,
                                     caffe_blob* bottom_diff, caffe_stream_t stream);

/* ------------------------------------------------------------------ the rest of the layer catalogue
   P:158 (Sec. 3.2): "nonlinearities like rectified linear and logistic ... element-wise operations
   ... losses like softmax and hinge".  Elementwise ops read and write every blob in its own memory
   order, so all blobs of a call must share shape, dtype (F32 or BF16) and layout; 16-byte aligned
   buffers (CAFFE_E_ALIGN otherwise).  n == 0 is a no-op.

   Sigmoid: top = 1/(1+e^-x); bottom_diff = top_diff * top * (1 - top), computed from the
   forward OUTPUT, so top may alias bottom (in place) and bottom_diff may alias top_diff. */
caffe_status caffe_sigmoid_forward(const caffe_blob* bottom, caffe_blob* top, caffe_stream_t stream);
caffe_status caffe_sigmoid_backward(const caffe_blob* top, const caffe_blob* top_diff, caffe_blob* bottom_diff,
                                    caffe_stream_t stream);

/* Eltwise over 2..CAFFE_ELTWISE_MAX_INPUTS inputs:
   SUM: top = sum_i coeff_i x_i (coeffs: host array of n_inputs floats, NULL = all 1; SUM only);
   PROD: top = prod_i x_i;  MAX: top = max_i x_i.
   Backward: SUM diff_i = coeff_i top_diff; PROD diff_i = top_diff * prod_{j!=i} x_j (no division);
   MAX: top_diff to the first input holding the maximum (strict '>' scan: ties go to the lowest i,
   S:249), 0 to the others.  inputs: host array of n_inputs blob pointers (SUM backward may pass NULL
   inputs); bottom_diffs: host array of n_inputs blob pointers, each overwritten (none may overlap an
   input or another diff).  Fewer than 2 inputs or > CAFFE_ELTWISE_MAX_INPUTS: CAFFE_E_PARAM;
   shape mismatch: CAFFE_E_SHAPE. */
#define CAFFE_ELTWISE_MAX_INPUTS 8
typedef enum { CAFFE_ELTWISE_PROD = 0, CAFFE_ELTWISE_SUM = 1, CAFFE_ELTWISE_MAX = 2 } caffe_eltwise_op;
caffe_status caffe_eltwise_forward(int32_t op, int32_t n_inputs, const caffe_blob* const* inputs, const float* coeffs,
                                   caffe_blob* top, caffe_stream_t stream);
caffe_status caffe_eltwise_backward(int32_t op, int32_t n_inputs, const caffe_blob* const* inputs, const float* coeffs,
                                    const caffe_blob* top_diff, caffe_blob* const* bottom_diffs, caffe_stream_t stream);

/* One-vs-all L1 hinge loss: y_nk = +1 if k == label_n else -1;
   loss (device F32 scalar) = (1/N) sum_{n,k} max(0, 1 - y_nk s_nk);
   score_diff (nullable) = -y_nk [1 - y_nk s_nk > 0] / N.  scores (N,K,1,1) F32/BF16; labels device
   int32[N].  The sum is in a fixed order (deterministic).  A label outside [0,K) is never
   used as an index: the loss and that row's diff are NaN. */
caffe_status caffe_hinge_loss(const caffe_blob* scores, const int32_t* labels, float* loss, caffe_blob* score_diff,
                              caffe_stream_t stream);

/* ------------------------------------------------------------------ solver (Sec. 3.4)
   Learning-rate schedules: FIXED lr = base_lr; STEP lr = base_lr * gamma^floor(iter /
   stepsize); INV lr = base_lr * (1 + gamma*iter)^-power (evaluated in FP64, rounded to F32).
   caffe_solver_state lives in DEVICE memory (caller-owned, zero-initialised = iteration 0) so a
   captured CUDA graph of the training step sees the current iteration on every replay:
     caffe_solver_begin: after the loss of this step is computed -- if *loss is not finite, sets
       `diverged` (sticky) and `diverged_iter` (the S:524 divergence guard); writes lr = lr_at(iter);
     caffe_sgd_update_solver: caffe_sgd_update with lr read from the state; does nothing once
       `diverged` is set (the parameters, momentum and BF16 copy keep their pre-step values);
     caffe_solver_end: iter += 1 unless diverged.
   The host reads the state after synchronising and aborts the loop on `diverged`. */
typedef enum { CAFFE_LR_FIXED = 0, CAFFE_LR_STEP = 1, CAFFE_LR_INV = 2 } caffe_lr_kind;
typedef struct { int32_t policy; float base_lr, gamma, power; int32_t stepsize; } caffe_lr_policy;
typedef struct {
    int64_t iter;          /* iterations completed */
    int64_t diverged_iter; /* iteration whose loss was non-finite (valid when diverged) */
    float lr;              /* learning rate of the current iteration (written by caffe_solver_begin) */
    float last_loss;       /* loss seen by the last caffe_solver_begin */
    int32_t diverged;
    int32_t reserved;
} caffe_solver_state;
caffe_status caffe_lr_at_iter(const caffe_lr_policy* policy, int64_t iter, float* lr /* host */);
caffe_status caffe_solver_begin(const caffe_lr_policy* policy, caffe_solver_state* state /* device */,
                                const float* loss /* device, nullable */, caffe_stream_t stream);
caffe_status caffe_solver_end(caffe_solver_state* state /* device */, caffe_stream_t stream);
caffe_status caffe_sgd_update_solver(float* w, const float* g, float* v, void* w_bf16, int64_t count,
                                     const caffe_solver_state* state /* device */, float momentum, float decay,
                                     float grad_scale, caffe_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CAFFE_B200_H_ */
