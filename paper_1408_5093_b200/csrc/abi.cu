// abi.cu -- the extern "C" boundary (include/caffe_b200.h): host-side validation, workspace
// planning and launch sequencing.  Every numerical step runs in the kernels of tc_gemm.cu,
// pack.cu and simple.cu; nothing here touches device data.
#include "../../include/caffe_b200.h"
#include "internal.h"
#include <algorithm>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using namespace cb;

// ------------------------------------------------------------------ instrumentation
namespace {
std::atomic<long long> g_launches{0};
struct ProfRec {
    cudaEvent_t a, b;
    double flops;
    int kind;
};
std::mutex g_pmu;
bool g_prof = false;
std::vector<ProfRec> g_recs;
std::vector<cudaEvent_t> g_evpool;
size_t g_evused = 0;
cudaEvent_t prof_event() {
    if (g_evused == g_evpool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        g_evpool.push_back(e);
    }
    return g_evpool[g_evused++];
}
}  // namespace
void cb::note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {

thread_local std::string g_err;

caffe_status fail(caffe_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}
caffe_status cuda_fail(cudaError_t e, const char* what) {
    return fail(CAFFE_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
#define CK(expr, what)                                     \
    do {                                                   \
        cudaError_t _e = (expr);                           \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

inline long long cnt(const caffe_shape4& s) { return (long long)s.n * s.c * s.h * s.w; }
inline size_t esize(caffe_dtype d) { return d == CAFFE_BF16 ? 2 : (d == CAFFE_U8 || d == CAFFE_I8) ? 1 : 4; }
inline size_t bytes_of(const caffe_blob* b) { return (size_t)cnt(b->shape) * esize(b->dtype); }
inline long long rup(long long a, long long b) { return (a + b - 1) / b * b; }
inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }
inline size_t align1k(size_t x) { return (x + 1023) & ~size_t(1023); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
inline bool nhwc(const caffe_blob* b) { return b->layout == CAFFE_NHWC; }
inline int isbf(const caffe_blob* b) { return b->dtype == CAFFE_BF16; }

L4 strides(const caffe_blob* b) {
    const caffe_shape4& s = b->shape;
    if (nhwc(b)) return L4{s.h * s.w * s.c, 1, s.w * s.c, s.c};
    return L4{s.c * s.h * s.w, s.h * s.w, s.w, 1};
}

caffe_status check_blob(const caffe_blob* b, const char* name, bool float_only = true) {
    if (!b) return fail(CAFFE_E_INVALID, "%s is NULL", name);
    if (!b->ptr && cnt(b->shape) != 0) return fail(CAFFE_E_INVALID, "%s->ptr is NULL", name);
    const caffe_shape4& s = b->shape;
    if (s.n < 0 || s.c < 0 || s.h < 0 || s.w < 0) return fail(CAFFE_E_SHAPE, "%s has a negative axis", name);
    if (s.n > 0 && (s.c == 0 || s.h == 0 || s.w == 0))
        return fail(CAFFE_E_SHAPE, "%s has a zero axis (%d,%d,%d,%d)", name, s.n, s.c, s.h, s.w);
    if (cnt(s) >= (1LL << 31)) return fail(CAFFE_E_SHAPE, "%s has >= 2^31 elements", name);
    if (b->layout != CAFFE_NCHW && b->layout != CAFFE_NHWC) return fail(CAFFE_E_INVALID, "%s has a bad layout %d", name, b->layout);
    if (float_only && b->dtype != CAFFE_F32 && b->dtype != CAFFE_BF16)
        return fail(CAFFE_E_DTYPE, "%s dtype must be F32 or BF16", name);
    if (!float_only && b->dtype != CAFFE_I32 && b->dtype != CAFFE_U8)
        return fail(CAFFE_E_DTYPE, "%s dtype must be I32 or U8", name);
    return CAFFE_OK;
}
bool overlap(const caffe_blob* a, const caffe_blob* b) {
    if (!a || !b || !a->ptr || !b->ptr) return false;
    const char* x = (const char*)a->ptr;
    const char* y = (const char*)b->ptr;
    return x < y + bytes_of(b) && y < x + bytes_of(a);
}
bool same_shape(const caffe_shape4& a, const caffe_shape4& b) {
    return a.n == b.n && a.c == b.c && a.h == b.h && a.w == b.w;
}

// ------------------------------------------------------------------ conv planning
struct Plan {
    int N, C, H, W, O, G, Cg, Og, kh, kw, sh, sw, ph, pw, OH, OW;
    int E, CH;             // operand element size, elements per 128-byte row
    bool s2d;
    int bh, bw, khp, kwp, php, pwp, Hp, Wp, Cge, Cgp, Ogp, taps;
};

caffe_status conv_validate(const caffe_conv_desc* d, caffe_shape4 bottom, int32_t O, Plan* p) {
    if (!d) return fail(CAFFE_E_INVALID, "desc is NULL");
    if (d->kernel_h < 1 || d->kernel_w < 1 || d->stride_h < 1 || d->stride_w < 1 || d->pad_h < 0 || d->pad_w < 0 ||
        d->group < 1)
        return fail(CAFFE_E_PARAM, "bad conv parameter (kernel %dx%d stride %dx%d pad %dx%d group %d)", d->kernel_h,
                    d->kernel_w, d->stride_h, d->stride_w, d->pad_h, d->pad_w, d->group);
    if (d->math != CAFFE_MATH_FP32 && d->math != CAFFE_MATH_TF32 && d->math != CAFFE_MATH_BF16)
        return fail(CAFFE_E_INVALID, "bad math mode %d", (int)d->math);
    if (bottom.c % d->group) return fail(CAFFE_E_PARAM, "channels %d not divisible by group %d", bottom.c, d->group);
    if (O < 1 || O % d->group) return fail(CAFFE_E_PARAM, "num_output %d not divisible by group %d", O, d->group);
    if (d->kernel_h > bottom.h + 2 * d->pad_h || d->kernel_w > bottom.w + 2 * d->pad_w)
        return fail(CAFFE_E_PARAM, "kernel %dx%d larger than padded input %dx%d (S:146)", d->kernel_h, d->kernel_w,
                    bottom.h + 2 * d->pad_h, bottom.w + 2 * d->pad_w);
    if (d->pad_h > 100 || d->pad_w > 100 || d->kernel_h > 100 || d->kernel_w > 100)
        return fail(CAFFE_E_PARAM, "kernel/pad larger than 100 not supported");
    Plan& q = *p;
    q.N = bottom.n; q.C = bottom.c; q.H = bottom.h; q.W = bottom.w; q.O = O; q.G = d->group;
    q.Cg = q.C / q.G; q.Og = O / q.G; q.kh = d->kernel_h; q.kw = d->kernel_w; q.sh = d->stride_h; q.sw = d->stride_w;
    q.ph = d->pad_h; q.pw = d->pad_w;
    q.OH = (q.H + 2 * q.ph - q.kh) / q.sh + 1;
    q.OW = (q.W + 2 * q.pw - q.kw) / q.sw + 1;
    q.E = d->math == CAFFE_MATH_TF32 ? 4 : 2;
    q.CH = 128 / q.E;
    q.s2d = q.sh > 1 || q.sw > 1;
    q.bh = q.s2d ? q.sh : 1; q.bw = q.s2d ? q.sw : 1;
    q.khp = (int)cdiv(q.kh, q.bh); q.kwp = (int)cdiv(q.kw, q.bw);
    q.php = q.s2d ? 0 : q.ph; q.pwp = q.s2d ? 0 : q.pw;
    q.Hp = q.s2d ? q.OH + q.khp - 1 : q.H;
    q.Wp = q.s2d ? q.OW + q.kwp - 1 : q.W;
    q.Cge = q.Cg * q.bh * q.bw;
    q.Cgp = (int)rup(q.Cge, q.CH);
    q.Ogp = (int)rup(q.Og, q.CH);
    q.taps = q.khp * q.kwp;
    return CAFFE_OK;
}

ConvGeom cgeom(const Plan& p) {
    return ConvGeom{p.N, p.C, p.H, p.W, p.O, p.kh, p.kw, p.sh, p.sw, p.ph, p.pw, p.G, p.OH, p.OW};
}
WGeom wgeom(const Plan& p) {
    return WGeom{p.O, p.G, p.Cg, p.Og, p.kh, p.kw, p.bh, p.bw, p.khp, p.kwp, p.Cgp, p.Ogp};
}

// An activation consumed by a TMA operand: either the caller's NHWC BF16 blob as-is, or a packed
// channels-last copy in workspace.  Group g's channels start at g*cpg; Ctot channels per pixel.
// A 64-channel operand block may run past its group's channels: those K positions meet zero
// weights (forward/data gradient) or produce discarded rows (weight gradient).
struct Operand {
    const void* ptr;
    int Ctot, cpg, H, W;
    bool packed;
    PackGeom pg;
};
int round_ch(int c, int E) { return (int)rup(c, 16 / E); }
bool can_use_direct(const caffe_blob* b, int Cg, int E, bool s2d) {
    return !s2d && E == 2 && b->dtype == CAFFE_BF16 && nhwc(b) && (b->shape.c * 2) % 16 == 0 && (Cg * 2) % 16 == 0 &&
           aligned16(b->ptr);
}
// X-like operand (conv forward input, wgrad input)
Operand plan_x(const caffe_blob* b, const Plan& p) {
    if (can_use_direct(b, p.Cg, p.E, p.s2d)) return Operand{b->ptr, p.C, p.Cg, p.H, p.W, false, {}};
    const int cpg = round_ch(p.Cge, p.E);
    return Operand{nullptr, p.G * cpg, cpg, p.Hp, p.Wp, true,
                   PackGeom{p.N, p.C, p.H, p.W, p.G, p.Cg, p.bh, p.bw, p.s2d ? p.ph : 0, p.s2d ? p.pw : 0, p.Hp, p.Wp,
                            cpg, p.G * cpg}};
}
// dY-like operand (conv backward inputs): O channels on the OH x OW grid, never s2d
Operand plan_dy(const caffe_blob* b, const Plan& p) {
    if (can_use_direct(b, p.Og, p.E, false)) return Operand{b->ptr, p.O, p.Og, p.OH, p.OW, false, {}};
    const int cpg = round_ch(p.Og, p.E);
    return Operand{nullptr, p.G * cpg, cpg, p.OH, p.OW, true,
                   PackGeom{p.N, p.O, p.OH, p.OW, p.G, p.Og, 1, 1, 0, 0, p.OH, p.OW, cpg, p.G * cpg}};
}
// conservative (always-packed) sizes used for workspace queries
size_t ws_x_max(const Plan& p) { return align1k((size_t)p.N * p.Hp * p.Wp * p.G * round_ch(p.Cge, p.E) * p.E); }
size_t ws_dy_max(const Plan& p) { return align1k((size_t)p.N * p.OH * p.OW * p.G * round_ch(p.Og, p.E) * p.E); }
size_t ws_wb(const Plan& p) { return align1k((size_t)p.O * p.taps * p.Cgp * p.E); }
size_t ws_wd(const Plan& p) { return align1k((size_t)p.G * p.Cge * p.taps * p.Ogp * p.E); }
size_t ws_t(const Plan& p) { return p.s2d ? align1k((size_t)p.N * p.Hp * p.Wp * p.G * p.Cge * 4) : 0; }
size_t ws_bias(const Plan& p) { return align1k((size_t)bias_grad_splits(p.N, p.O, p.OH * p.OW) * p.O * 4); }

caffe_status pack_if(const Operand& o, const caffe_blob* src, void* dst, int E, cudaStream_t s) {
    if (!o.packed) return CAFFE_OK;
    CK(pack_act(src->ptr, isbf(src), strides(src), nhwc(src), dst, E, o.pg, s), "pack activations");
    return CAFFE_OK;
}

int choose_bn(int n) {
    if (n <= 256) return (int)rup(n, 16);
    const int t = (int)cdiv(n, 256);
    return (int)rup(cdiv(n, t), 16);
}
// CTA pairs (M=256 tiles, cta_group::2) whenever the pair-tiles still fill every SM pair once.
int g_max_ctas = 0;  // CAFFE_TUNE_MAX_CTAS: cap on the persistent tensor-core grid (0 = one CTA per SM)
int g_force_cg = 0;   // caffe_set_tuning(CAFFE_TUNE_CTA_PAIR, 1|2) overrides the automatic choice
int g_mma_spin = 0;   // CAFFE_TUNE_MMA_SPIN (polling measured slower: it steals issue slots from the epilogue)
int pick_cg(long long M, int ntiles_x_groups, int E) {
    if (E != 2) return 1;
    if (g_force_cg == 1 || g_force_cg == 2) return g_force_cg;
    const long long pair_units = cdiv(M, 256) * ntiles_x_groups;
    return pair_units >= num_sms() / 2 ? 2 : 1;
}
int pow2ceil(int x) {
    int p = 32;
    while (p < x) p <<= 1;
    return p;
}
void finish_args(TcArgs& a, int bstage) {
    a.b_stage_bytes = bstage;
    const int macc = a.macc > 1 ? a.macc : 1;
    const int stage = macc * 16384 + bstage;
    a.stages = (200 * 1024) / stage;
    if (a.stages > 8) a.stages = 8;
    a.acc_stride = pow2ceil(a.BN);
    // two accumulator buffers when they fit in the 512 TMEM columns, else one
    a.tmem_cols = 2 * macc * a.acc_stride <= 512 ? 2 * macc * a.acc_stride : macc * a.acc_stride;
    if (a.tmem_cols < 32) a.tmem_cols = 32;
    a.tmem_cols = pow2ceil(a.tmem_cols);
    a.units = a.m_tiles * a.n_tiles * a.groups * a.splits;
}
// TMA-store epilogue for a row-major output [rows][ld] (cols valid): only plain stores (beta == 0),
// whole 128-byte column boxes inside each tile, 16-byte aligned rows.  Call after finish_args.
int g_tma_store = 1;   // CAFFE_TUNE_TMA_STORE
void enable_tma_store(TcLaunch& L, void* out, int esz, long long cols, long long rows, long long ld, bool groups_ok) {
    TcArgs& a = L.args;
    const int cw = 128 / esz;
    if (!g_tma_store || a.beta != 0.f || !groups_ok || a.BN % cw != 0 || (ld * esz) % 16 != 0 ||
        (reinterpret_cast<uintptr_t>(out) & 15) != 0 || (a.macc > 1))
        return;
    if (!encode_store_2d(&L.mapC, esz, out, (uint64_t)cols, (uint64_t)rows, (uint64_t)ld)) return;
    a.tma_store = 1;
    const int macc = a.macc > 1 ? a.macc : 1;
    const int stage = macc * 16384 + a.b_stage_bytes;
    a.stages = std::min(8, (200 * 1024 - 33 * 1024) / stage);
}
// Row-staged coalesced epilogue (epi_store_rows) for s_c == 1 outputs with beta 0: 16-byte aligned
// rows, group column offsets and N; TMEM slots wide enough for whole 128-byte column chunks.
int g_rows_epi = 0;   // CAFFE_TUNE_ROWS_EPILOGUE (off: adds epilogue instructions where the epilogue is the
                      // bottleneck -- conv1 forward 106 -> 149 us; no gain elsewhere)
void enable_rows_epilogue(TcArgs& a) {
    const bool ok = g_rows_epi && !a.tma_store && !a.relu_top && a.s_c == 1 && a.beta == 0.f && a.out_bf16 && a.BN <= 128 &&
                    a.BN % 8 == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0 && (a.s_p * 2) % 16 == 0 &&
                    (a.s_n * 2) % 16 == 0 && ((long long)a.col_g * 2) % 16 == 0 && a.N % 8 == 0;
    a.rows_epi = ok ? 1 : 0;
}
void set_out(TcArgs& a, const caffe_blob* b) {
    // m = image * P + pixel;  column = output channel
    const caffe_shape4& s = b->shape;
    if (nhwc(b)) { a.s_n = (long long)s.h * s.w * s.c; a.s_c = 1; a.s_p = s.c; }
    else { a.s_n = (long long)s.c * s.h * s.w; a.s_c = (long long)s.h * s.w; a.s_p = 1; }
    a.P = s.h * s.w;
    a.out = b->ptr;
    a.out_bf16 = isbf(b);
}
void finish_rows_epilogue(TcArgs& a) {
    enable_rows_epilogue(a);
    if (a.rows_epi) {   // 16 KB of staging: keep the total under the 227 KB limit
        const int macc = a.macc > 1 ? a.macc : 1;
        const int stage = macc * 16384 + a.b_stage_bytes;
        const int budget = (a.tma_store ? 167 : 200) * 1024 - 35 * 1024;
        a.stages = std::min(a.stages, std::max(2, budget / stage));
    }
}

struct WgradSplit {
    int m_tiles, n_tiles, BN, splits, kb_per, kblocks;
    int macc, m_groups;   // accumulators (M tiles) per work unit and the resulting unit rows
};
int g_wgrad_macc = 0;     // CAFFE_TUNE_WGRAD_MACC: 0 = automatic, 1..4 forced
WgradSplit wgrad_split(const Plan& p) {
    WgradSplit w;
    const int nchunks = p.taps * (p.Cgp / p.CH);
    const int chunks_per_tile = 128 / p.CH;
    w.m_tiles = (int)cdiv(nchunks, chunks_per_tile);
    w.BN = choose_bn(p.Og);
    w.n_tiles = (int)cdiv(p.Og, w.BN);
    w.kblocks = (int)cdiv((long long)p.N * p.OH * p.OW, p.CH);
    // Several M tiles per unit stage dY (the B operand, re-read once per unit) once for all of
    // them: the most accumulators that fit the 512 TMEM columns (single-buffered when two sets do
    // not fit -- measured faster than fewer, double-buffered accumulators: the units are long)
    // with stages still 3 deep in shared memory.
    const int accs = pow2ceil(w.BN);
    const int bstage = (int)cdiv(w.BN, p.CH) * p.CH * 128;
    w.macc = 1;
    if (g_wgrad_macc >= 1) {
        w.macc = g_wgrad_macc;
        while (w.macc > 1 && (w.macc * accs > 512 || (200 * 1024) / (w.macc * 16384 + bstage) < 2)) w.macc--;
    } else {
        for (int m = 2; m <= 4; m++) {
            if (m * accs > 512 || (200 * 1024) / (m * 16384 + bstage) < 3) break;
            w.macc = m;
        }
    }
    if (w.macc > w.m_tiles) w.macc = w.m_tiles;
    // (TF32 takes the same choice: tools/tf32_probe.py, batch 256, conv2-5 weight gradients
    // 1271/468/389/350 us with one accumulator, 1060/370/312/282 us with 2-4)
    w.m_groups = (int)cdiv(w.m_tiles, w.macc);
    // Split the pixel reduction so that (tiles x splits) work units fill the SMs in whole waves:
    // maximise wave efficiency x split balance x kb/(kb + 2) (per-unit prologue/epilogue cost).
    const int tiles = w.m_groups * w.n_tiles * p.G;
    const int sms = 148;
    double best = -1.0;
    w.kb_per = w.kblocks;
    w.splits = 1;
    for (int s = 1; s <= 1024 && s <= w.kblocks; s++) {
        const int kb_per = (int)cdiv(w.kblocks, s);
        if (kb_per < 4 && s > 1) break;
        const int ss = (int)cdiv(w.kblocks, kb_per);
        const long long units = (long long)tiles * ss;
        const double wave = (double)units / (double)(cdiv(units, sms) * sms);
        const double bal = (double)w.kblocks / ((double)ss * kb_per);
        const double eff = wave * bal * kb_per / (kb_per + 2.0);
        if (eff > best + 1e-9) {
            best = eff;
            w.kb_per = kb_per;
            w.splits = ss;
        }
    }
    return w;
}
// ---- halo-tiled weight gradient (tc_halo.cu, A_HALO_MN): single 64-channel block layers
int g_halo = 0;   // CAFFE_TUNE_HALO: 0 = automatic, 1 = off (im2col tiles), 2 = wherever it applies
struct WgHalo {
    bool use;
    int Wt, TH, rows, tpi, total, ksteps, cblocks;  // tile geometry (output tile = TH rows x Wt columns)
    int BN, n_tiles, nch, acc_stride, macc, pairs, mgroups, splits, kb_per, slot, bchunk, stages;
};
// CAFFE_TUNE_IP_FWD_SMALL_BN: N tile of inner-product forwards with <= 1024 outputs (fc8: 8 N tiles x
// 9 splits instead of 4 x 16 -- 9.4 instead of 16.8 MB of partials; GEMM + reduce 16.2 -> 12.4-12.8 us
// alone, tools/fc8_probe.py; the forward runs alone on the GPU, so this is step time; the 4-run step
// A/B was within its noise)
int g_ip_fwd_small_bn = 128;
int g_ip_max_splits = 0;   // CAFFE_TUNE_IP_MAX_SPLITS: cap on the inner-product split-K factor (0 = none)
int g_wgrad_bn = 0;   // CAFFE_TUNE_WGRAD_BN: N tile of the halo weight gradient (0 = automatic)
WgHalo wgrad_halo_plan(const Plan& p) {
    WgHalo h;
    memset(&h, 0, sizeof h);
    if (p.E != 2 || g_halo == 1 || p.taps < 2) return h;
    h.Wt = p.OW + p.kwp - 1;
    if (h.Wt > 256) return h;
    // tile = TH whole output rows (K rows padded to 16): the TH with the fewest idle K rows, up to 256
    // rows (13x13 maps: one whole image per tile, 81% useful rows instead of 66% with 8-row tiles)
    // (tiles of >= 112 rows -- or the whole image -- so the staged window and the per-tile barrier
    // traffic stay amortised; ties go to the larger tile)
    double best = -1.0;
    const int max_rows = g_halo == 3 ? 128 : 256;   // CAFFE_TUNE_HALO 3: tiles of <= 128 pixel rows
    const long long min_rows = std::min<long long>(112, rup((long long)p.OH * h.Wt, 16));
    for (int th = 1; th <= p.OH && th * h.Wt <= max_rows; th++) {
        if (rup((long long)th * h.Wt, 16) < min_rows) continue;
        const int tpi = (int)cdiv(p.OH, th);
        const double eff = (double)p.OH * p.OW / ((double)tpi * rup((long long)th * h.Wt, 16));
        if (eff >= best - 1e-9) { best = eff; h.TH = th; }
    }
    if (h.TH == 0) return h;
    if (g_halo < 2 && (p.taps < 4 || best < 0.75)) return h;
    h.tpi = (int)cdiv(p.OH, h.TH);
    h.ksteps = (int)cdiv((long long)h.TH * h.Wt, 16);
    h.rows = h.TH + p.khp - 1;
    h.total = p.N * h.tpi;
    h.cblocks = p.Cgp / 64;
    h.BN = choose_bn(p.Og);
    // several channel blocks (the 13x13 layers): every tap of a channel block in one unit -- 5
    // accumulators of <= 96 columns -- so the staged window serves all taps.  CAFFE_TUNE_WGRAD_BN 1
    // takes the widest N tile of <= 192 columns instead (an MMA reads a 4 KB A tile per K step, so
    // narrow N is shared-memory bound; wider tiles fit fewer taps per unit and restage the window):
    // faster alone (tools/wgrad_probe.py, batch 256, us: conv3 92.4 -> 86.9, conv4 72.8 -> 66.7,
    // conv5 59.6 -> 51.7) but slower in the three-stream step (tools/sched_sweep.py, same box:
    // 1.51-1.54 -> 1.57-1.62 ms/step), so off by default
    if (h.cblocks > 1 && g_wgrad_bn == 2) {   // <= 96 columns, but 128 rather than 64
        if (p.Og % 96 == 0) h.BN = 96;
        else if (p.Og % 128 == 0) h.BN = 128;
        else if (p.Og % 64 == 0) h.BN = 64;
    } else if (h.cblocks > 1 && g_wgrad_bn != 1) {
        if (p.Og % 96 == 0) h.BN = 96;
        else if (p.Og % 64 == 0) h.BN = 64;
    } else if (h.cblocks > 1) {
        if (p.Og % 192 == 0) h.BN = 192;
        else if (p.Og % 128 == 0) h.BN = 128;
        else if (p.Og % 96 == 0) h.BN = 96;
        else if (p.Og % 64 == 0) h.BN = 64;
    }
    if (g_wgrad_bn > 2 && g_wgrad_bn % 16 == 0 && g_wgrad_bn <= 256) h.BN = std::min(g_wgrad_bn, (int)rup(p.Og, 16));
    if (h.BN > 256) return h;
    h.n_tiles = (int)cdiv(p.Og, h.BN);
    h.nch = (int)cdiv(h.BN, 64);
    h.acc_stride = (int)rup(h.BN, 32);
    const int mmax = std::min(5, 512 / h.acc_stride);
    h.pairs = (int)cdiv(p.taps, 2);
    h.mgroups = (int)cdiv(h.pairs, mmax);
    h.macc = (int)cdiv(h.pairs, h.mgroups);          // largest balanced group
    const int krows = h.ksteps * 16;
    const int need_rows = std::max(h.rows * h.Wt, krows + (p.khp - 1) * h.Wt + (p.kwp - 1));
    h.slot = (int)rup((long long)need_rows * 128, 1024);
    h.bchunk = (int)rup((long long)krows * 128, 1024);   // K rows x 64 channels
    const int stage = h.slot + h.nch * h.bchunk;
    h.stages = std::min(8, (232448 - 1024 - 2048 - 1024) / stage);
    if (h.stages < 2) return h;
    const int base = p.G * h.n_tiles * h.mgroups * h.cblocks;   // units per pixel split
    int sp = std::max(1, 148 / base);
    sp = std::min(sp, std::max(1, h.total / 4));
    h.kb_per = (int)cdiv(h.total, sp);
    h.splits = (int)cdiv(h.total, h.kb_per);
    h.use = true;
    return h;
}
size_t ws_partial(const Plan& p) {
    WgradSplit w = wgrad_split(p);
    size_t b = (size_t)w.m_tiles * w.n_tiles * p.G * w.splits * w.BN * 128 * 4;
    const WgHalo h = wgrad_halo_plan(p);
    if (h.use) b = std::max(b, (size_t)h.splits * p.G * h.cblocks * h.pairs * h.n_tiles * h.BN * 128 * 4);
    return align1k(b);
}

size_t conv_ws(const Plan& p, int pass, caffe_math m) {
    if (pass == CAFFE_PASS_BACKWARD_WEIGHT) {
        if (m == CAFFE_MATH_FP32) return ws_bias(p);
        return ws_x_max(p) + ws_dy_max(p) + ws_partial(p) + ws_bias(p);
    }
    if (m == CAFFE_MATH_FP32) return 0;
    if (pass == CAFFE_PASS_FORWARD) return ws_x_max(p) + ws_wb(p);
    return ws_dy_max(p) + ws_wd(p) + ws_t(p);
}

caffe_status check_ws(void* ws, size_t have, size_t need) {
    if (need == 0) return CAFFE_OK;
    if (!ws || have < need)
        return fail(CAFFE_E_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws ? have : (size_t)0);
    if ((reinterpret_cast<uintptr_t>(ws) & 1023) != 0) return fail(CAFFE_E_ALIGN, "workspace must be 1024-byte aligned");
    return CAFFE_OK;
}

// kind: 0 = convolution pass, 1 = inner product; flops = algorithmic FLOPs of the call
// ---- halo-tiled stride-1 convolution (tc_halo.cu)
struct HaloGeom {
    int Hi, Wi, Ho, Wo, kh, kw, pad_h, pad_w;   // stride-1 geometry of the pass (input -> output)
};
// Tile shape and whether the halo form is used: halo_wt = Wo + kw - 1 columns, halo_th = 128 / halo_wt
// output rows per 128-row tile.  Automatic use needs >= 4 taps and >= 75% useful accumulator rows
// (CaffeNet conv1/conv2: 84% / 81%; the 13x13 layers reach only 66% and stay on im2col tiles).
static bool halo_applies(int E, const HaloGeom& h) {
    if (E != 2 || g_halo == 1) return false;
    const int wt = h.Wo + h.kw - 1;
    if (wt > 128 || h.Ho < 1) return false;
    const int th = 128 / wt;
    if (th + h.kh - 1 > 256) return false;
    if (g_halo >= 2) return true;
    const int tpi = (h.Ho + th - 1) / th;
    const double eff = (double)h.Ho * h.Wo / (tpi * 128.0);
    return h.kh * h.kw >= 4 && eff >= 0.75;
}
// Stacked halo tiles (TcArgs::stk) for same-size stride-1 convolutions with odd kernels and
// centred padding (CaffeNet conv3-5 forward and data gradient: 3x3/pad 1 on 13x13), whose maps
// are too small for whole-row halo tiles (66% useful rows) and whose per-tap im2col tiles stream
// every activation 9x from L2: rows W + pad_w wide and images H + pad_h tall in one pixel sequence,
// 86% useful rows for 13x13.  CAFFE_TUNE_HALO_STACKED: 0 off, 1 (default) where whole-row halo tiles
// do not apply, 2 wherever the geometry allows.
int g_halo_stacked = 1;
static bool stacked_geom(const HaloGeom& h) {
    return h.Ho == h.Hi && h.Wo == h.Wi && (h.kh & 1) && (h.kw & 1) && h.pad_h == (h.kh - 1) / 2 &&
           h.pad_w == (h.kw - 1) / 2 && h.kh * h.kw >= 4 && h.Wi + h.pad_w <= 256 && h.Wo >= 4;
}
// Automatic use only with N tiles of <= 128 columns (two accumulators per CTA share each weight
// tile): measured on CaffeNet (us, per-tap im2col -> stacked) conv5 forward 46.2 -> 39.7, but
// conv3/conv4 forward 60.3/48.1 -> 63.2/51.0 and the 192/256-column data gradients 59.0/48.4/35.1 ->
// 67.5/52.2/38.8 (one accumulator per CTA: every weight tile feeds a single 128-pixel tile).
static bool stacked_applies(int E, const HaloGeom& h, int BN) {
    if (E != 2 || g_halo == 1 || g_halo_stacked == 0 || !stacked_geom(h)) return false;
    if (g_halo_stacked >= 2) return true;
    return !halo_applies(E, h) && BN <= 128;
}
// N tile of a halo/stacked pass: CAFFE_TUNE_HALO_STACKED 4 splits the columns of stacked-geometry
// passes into tiles of <= 128 (two accumulators per CTA, double-buffered: conv3 384 -> 3 x 128,
// conv4/conv5 data gradient 192 -> 2 x 96)
static int halo_bn(int n, const HaloGeom& h) {
    if (g_halo_stacked == 4 && stacked_geom(h) && !halo_applies(2, h) && n > 128) {
        const int t = (int)cdiv(n, 128);
        return (int)rup(cdiv(n, t), 16);
    }
    return choose_bn(n);
}
// Fills the halo fields of L (A map over the channels-last operand `aptr` [N][Hi][Wi][Ctot]) after
// the caller has set BN, N, n_tiles, groups, b_row_g, a_cpg, a_cblocks and the epilogue.
int g_halo_ktrim = 1;   // CAFFE_TUNE_HALO_KTRIM
int g_halo_merge = 0;   // CAFFE_TUNE_HALO_MERGE (bit-identical; measured no faster: conv1 forward 110.8 vs
                        // 110.7 us with its pack, tools/merge_probe.py; step 1.50-1.52 vs 1.52-1.53 ms)
int g_halo_btaps = 0;   // CAFFE_TUNE_HALO_BTAPS
static bool halo_setup(TcLaunch& L, const HaloGeom& h, const void* aptr, int Ctot, int N) {
    TcArgs& a = L.args;
    L.amode = A_HALO_K; L.bmode = B_TILED_K; L.epi = EPI_STRIDED; L.esz = 2;
    a.halo_kh = h.kh; a.a_kw = h.kw;
    a.a_pad_h = h.pad_h; a.a_pad_w = h.pad_w;
    a.out_h = h.Ho; a.out_w = h.Wo;
    a.stk = stacked_applies(2, h, a.BN) ? 1 : 0;
    if (a.stk) {
        a.stk_wt = h.Wi + h.pad_w; a.stk_hs = h.Hi + h.pad_h; a.stk_nimg = N;
        a.stk_off = a.stk_wt - 1;
        a.halo_wt = a.stk_wt;             // tap (i, j) shift = i*stk_wt + j rows
        a.halo_th = 1; a.halo_rows = 1; a.tiles_per_img = 1;
        const int r_last = a.stk_off + 127 + (h.kh - 1) * a.stk_wt + (h.kw - 1);
        a.stk_nb = (r_last + a.stk_wt) / a.stk_wt;   // ceil((r_last + 1) / wt)
        a.halo_slot = (int)rup((long long)(a.stk_off + a.stk_nb * a.stk_wt) * 128, 1024);
        a.total_tiles = (int)cdiv((long long)N * a.stk_hs * a.stk_wt, 128);
        if (!encode_tiled_4d(&L.mapA, 2, aptr, Ctot, h.Wi, h.Hi, N, 64, (uint32_t)a.stk_wt, 1)) return false;
    } else {
        a.halo_wt = h.Wo + h.kw - 1;
        a.halo_th = 128 / a.halo_wt;
        a.halo_rows = a.halo_th + h.kh - 1;
        a.tiles_per_img = (h.Ho + a.halo_th - 1) / a.halo_th;
        a.total_tiles = N * a.tiles_per_img;
        const int need_rows = std::max(a.halo_rows * a.halo_wt, (h.kh - 1) * a.halo_wt + (h.kw - 1) + 128);
        a.halo_slot = (int)rup((long long)need_rows * 128, 1024);
        if (!encode_tiled_4d(&L.mapA, 2, aptr, Ctot, h.Wi, h.Hi, N, 64, (uint32_t)a.halo_wt, (uint32_t)a.halo_rows))
            return false;
    }
    // CTA pairs when the B tile splits into 8-row halves and there is enough work for every pair
    L.cg = 1;
    if ((a.BN / 2) % 8 == 0 &&
        (g_force_cg == 2 || (g_force_cg == 0 && (long long)a.total_tiles * a.n_tiles * a.groups >= 4LL * num_sms())))
        L.cg = 2;
    a.acc_stride = pow2ceil(a.BN);
    a.a_stages = 2;
    a.macc = 1;
    if (2 * 2 * a.acc_stride <= 512 && a.a_stages * 2 * a.halo_slot <= 140 * 1024) a.macc = 2;
    // CAFFE_TUNE_HALO_STACKED 3: stacked tiles of up to 256 columns also take two accumulators per
    // CTA (each weight tile feeds 2 x 128 pixels; the 512 TMEM columns then hold one set, so the
    // epilogue of a unit does not overlap the next unit's MMAs)
    if (a.stk && g_halo_stacked >= 3 && a.macc == 1 && a.acc_stride == 256 &&
        a.a_stages * 2 * a.halo_slot <= 140 * 1024)
        a.macc = 2;
    // (a deeper A ring for stacked tiles -- 3 or 4 stages -- measured no faster: 2 stages kept)
    // CAFFE_TUNE_HALO_MERGE: with two accumulators per CTA on whole-row tiles, the CTA takes two
    // consecutive row blocks of one image and stages ONE window of 2*halo_th + kh - 1 rows for both
    // (conv1: 6 instead of 2 x 4 input rows per stage), three stages deep where they fit; off by
    // default -- conv1's forward is bound by its output stores, not by the staging of its windows
    a.a_merge = 0;
    if (g_halo_merge && a.macc == 2 && !a.stk && a.tiles_per_img % 2 == 0) {
        const int mrows = 2 * a.halo_th + h.kh - 1;
        const int need = std::max(mrows * a.halo_wt, (h.kh - 1 + a.halo_th) * a.halo_wt + (h.kw - 1) + 128);
        const int mslot = (int)rup((long long)need * 128, 1024);
        const int st = 3LL * mslot <= 140 * 1024 ? 3 : 2;
        if ((long long)st * mslot <= 140 * 1024 &&
            encode_tiled_4d(&L.mapA, 2, aptr, Ctot, h.Wi, h.Hi, N, 64, (uint32_t)a.halo_wt, (uint32_t)mrows)) {
            a.a_merge = 1;
            a.halo_rows = mrows;
            a.halo_slot = mslot;
            a.a_stages = st;
        }
    }
    a.b_stage_bytes = a.BN / L.cg * 128;
    long long budget = 232448 - 512 - 2048 - 1024 - (long long)a.a_stages * (a.a_merge ? 1 : a.macc) * a.halo_slot;
    // TMA tensor-store epilogue (specialised-epilogue launches): the unit's tiles are staged in
    // shared memory as boxes of cw channels x Wo pixels x halo_th rows and leave through mapC
    a.tma_store = 0;
    // CAFFE_TUNE_HALO_EPI_GROUPS: the first layer's 96 output columns as three epilogue groups of 32
    // (first layer, 96 columns: default 3 -- conv1 forward 78.4 -> 71.8 us, 4 groups 73.8 us; the
    // 128-column passes of conv2 / conv5 forward measured slower with 4 groups of 32: 93.7 -> 94.9,
    // 40.5 -> 42.4 us -- their MMAs, not the epilogue, bound them)
    a.epi_groups = 2;
    if (a.BN == 96 && a.k_last == 3 && a.a_cblocks == 1)
        a.epi_groups = g_halo_epi_groups == 0 ? 3 : g_halo_epi_groups;
    const int epc = halo_fast_epc(a, L.cg);
    if (epc > 0 && cb::g_halo_tma_store && !a.stk && a.epi_groups == 2) {
        const int cwl = epc % 64 == 0 ? 6 : epc % 32 == 0 ? 5 : epc % 16 == 0 ? 4 : 0;
        const int cw = cwl ? 1 << cwl : epc;
        const int align = cwl ? 16 * cw : 128;   // the swizzle pattern repeats every 8 rows
        if (cwl > 0 || (epc / 8) % 2 == 1) {
            const int chunk = (int)rup((long long)a.halo_th * h.Wo * cw * 2, align);
            const int tile = (int)rup((long long)(a.BN / cw) * chunk, 1024);
            if ((long long)a.macc * tile <= 64 * 1024 &&
                encode_store_4d(&L.mapC, 2, a.out, (int)a.s_p, h.Wo, h.Ho, N, a.s_p, a.s_n, (uint32_t)cw,
                                (uint32_t)h.Wo, (uint32_t)a.halo_th, cwl ? cw * 2 : 0)) {
                a.tma_store = 1;
                a.st_cw = cwl;
                a.st_chunk_bytes = chunk;
                a.st_tile_bytes = tile;
                budget -= (long long)a.macc * tile + 1024;
            }
        }
    }
    // weights resident in shared memory when the whole filter (this CTA's half) fits: staged once
    // per kernel instead of once per unit (the first layer: 9 taps x 6 KB)
    const long long nb = (long long)h.kh * h.kw * a.a_cblocks;
    // coalesced stores of the specialised epilogue (per-warp transpose through shared memory), when
    // the staging fits beside resident weights -- the first layer, whose 148.7 MB output bounds it
    // (conv1 forward 81.7 -> 78.5 us; with a streamed B ring the staging costs B stages instead:
    // conv2 forward 92.4 -> 96.0 us)
    a.epi_coal = 0;
    if (epc > 0 && !a.tma_store && cb::g_halo_coal && a.groups == 1 && a.n_tiles == 1 && nb <= 24 &&
        nb * a.b_stage_bytes <= budget - (long long)halo_coal_bytes(a) - 1024) {
        a.epi_coal = 1;
        budget -= (long long)halo_coal_bytes(a) + 1024;
    }
    a.b_resident = 0;
    a.b_taps = 1;
    if (a.groups == 1 && a.n_tiles == 1 && nb <= 24 && nb * a.b_stage_bytes <= budget) {
        a.b_resident = 1;
        a.stages = (int)nb;
    } else {
        // CAFFE_TUNE_HALO_BTAPS: weight tiles per B stage (0 = automatic: 2 for tiles of <= 32 rows
        // per CTA, whose MMAs are short enough for the issue loop to matter)
        // compiled: 5 taps per stage for the specialised 24-column epilogue instance (conv2's data
        // gradient, 5x5 filter) when >= 4 stages still fit; 1 elsewhere
        const int epc_b = halo_fast_epc(a, L.cg);
        const int want = g_halo_btaps > 0 ? g_halo_btaps : 5;
        if (want == 5 && epc_b == 24 && a.k_last != 3 && (h.kh * h.kw) % 5 == 0 && budget / (5LL * a.b_stage_bytes) >= 4)
            a.b_taps = 5;
        a.b_stage_bytes *= a.b_taps;
        a.stages = (int)std::min<long long>(24, budget / a.b_stage_bytes);
    }
    if (a.stages < 2) return false;
    const int cols = (2 * a.macc * a.acc_stride <= 512 ? 2 : 1) * a.macc * a.acc_stride;
    a.tmem_cols = pow2ceil(cols < 32 ? 32 : cols);
    const int tgroups = (a.total_tiles + a.macc * L.cg - 1) / (a.macc * L.cg);
    a.units = a.groups * a.n_tiles * tgroups;
    a.m_tiles = tgroups; a.splits = 1;
    return true;
}

// Data gradient with a filter row's taps in the MMA's N (tc_halo_jn_kernel, A_HALO_JN): after
// halo_setup, for whole-row halo tiles of compiled (kh, kw, channels per group) shapes with 64-channel
// blocks of output channels, BF16 channels-last output, beta 0 and no ReLU gate (CaffeNet conv2).
// CAFFE_TUNE_HALO_JN: 1 (default) where it applies, 0 = the per-tap halo kernel.
int g_halo_jn = 1;
static bool jn_setup(TcLaunch& L, const Plan& p, const caffe_blob* bottom_diff, const caffe_blob* relu_top, float beta,
                     const void* WD) {
    TcArgs& a = L.args;
    if (!g_halo_jn || a.stk || a.a_merge || relu_top || beta != 0.f || !isbf(bottom_diff) || !nhwc(bottom_diff) || p.s2d) return false;
    if (!tc_halo_jn_compiled(p.khp, p.kwp, p.Cge) || p.Cge != p.Cg || p.Og % 64 != 0 || p.Ogp != p.Og) return false;
    if (a.s_p % 8 || a.s_n % 8 || a.col_g % 8 || (reinterpret_cast<uintptr_t>(a.out) & 15)) return false;
    if (num_sms() / 2 < p.G) return false;
    TcArgs t = a;
    t.a_stages = 2;
    if (tc_halo_jn_smem_bytes(t, p.khp, p.kwp, p.Cge) > 232448) return false;
    CUtensorMap mb;
    // WD [G*Cge rows][taps][Ogp] as a 4-D tensor (o, tap, row, 1): one box = 64 o x kw taps x Cge/2 rows
    if (!encode_tiled_4d(&mb, 2, WD, p.Ogp, p.taps, p.G * p.Cge, 1, 64, (uint32_t)p.kwp, (uint32_t)(p.Cge / 2)))
        return false;
    L.mapB = mb;
    L.amode = A_HALO_JN;
    L.cg = 2;
    a.a_stages = 2;
    a.macc = 1;
    a.acc_stride = 256;
    a.tmem_cols = 512;
    a.units = a.groups * (int)cdiv(a.total_tiles, 2);
    a.BN = p.kwp * p.Cge;
    return true;
}

caffe_status run_tc(TcLaunch& L, cudaStream_t s, double flops, int kind) {
    if (L.cg < 1) L.cg = 1;
    if (L.epi == EPI_STRIDED && L.amode != A_HALO_MN) {
        if (L.amode == A_HALO_K) {
            L.args.rows_epi = 0;   // the halo kernel splits its columns over two epilogue warp groups
        } else {
            finish_rows_epilogue(L.args);
        }
    }
    L.args.spin = g_mma_spin;
    int slots = num_sms() / L.cg;                        // CTAs (or CTA pairs) resident at once
    if (g_max_ctas > 0 && g_max_ctas / L.cg < slots)      // CAFFE_TUNE_MAX_CTAS: more units per CTA
        slots = g_max_ctas / L.cg > 0 ? g_max_ctas / L.cg : 1;
    L.grid = (L.args.units < slots ? L.args.units : slots) * L.cg;
    if (L.amode == A_HALO_JN) {   // each CTA pair serves one group: a multiple of `groups` pairs
        const int G = L.args.groups;
        int pairs = L.grid / 2;
        if (pairs < G) pairs = G;
        pairs -= pairs % G;
        L.grid = pairs * 2;
    }
    static const bool dbg = getenv("CAFFE_DEBUG_TC") != nullptr;   // launch-plan trace (development aid)
    if (dbg)
        fprintf(stderr, "tc amode %d bmode %d epi %d cg %d units %d grid %d BN %d macc %d stages %d kblocks %d "
                        "kb/split %d splits %d M %d N %d waves %.2f\n",
                L.amode, L.bmode, L.epi, L.cg, L.args.units, L.grid, L.args.BN, L.args.macc, L.args.stages,
                L.args.kblocks, L.args.kb_per_split, L.args.splits, L.args.M, L.args.N,
                (double)L.args.units / (L.grid / L.cg));
    ProfRec rec{nullptr, nullptr, flops, kind};
    if (g_prof) {
        std::lock_guard<std::mutex> lk(g_pmu);
        rec.a = prof_event();
        rec.b = prof_event();
        cudaEventRecord(rec.a, s);
    }
    cudaError_t e = L.amode == A_HALO_K    ? tc_halo_launch(L, s)
                    : L.amode == A_HALO_MN ? tc_halo_wgrad_launch(L, s)
                    : L.amode == A_HALO_JN ? tc_halo_jn_launch(L, s)
                                           : tc_launch(L, s);
    if (g_prof) {
        cudaEventRecord(rec.b, s);
        std::lock_guard<std::mutex> lk(g_pmu);
        g_recs.push_back(rec);
    }
    if (e != cudaSuccess) return cuda_fail(e, "tcgen05 GEMM launch");
    return CAFFE_OK;
}
double conv_flops(const Plan& p) { return 2.0 * p.N * p.O * p.OH * p.OW * (double)p.Cg * p.kh * p.kw; }

}  // namespace

// ====================================================================== exported
extern "C" {

int32_t caffe_abi_version(void) { return CAFFE_ABI_VERSION; }
const char* caffe_last_error(void) { return g_err.c_str(); }
int64_t caffe_launch_count(void) { return g_launches.load(); }

caffe_status caffe_profiler_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_pmu);
    if (on) {
        g_recs.clear();
        g_evused = 0;
    }
    g_prof = on != 0;
    return CAFFE_OK;
}

caffe_status caffe_profiler_read(int32_t kind, double* ms, double* flops, int64_t* launches) {
    if (!ms || !flops || !launches) return fail(CAFFE_E_INVALID, "NULL output pointer");
    std::lock_guard<std::mutex> lk(g_pmu);
    double t = 0.0, f = 0.0;
    int64_t n = 0;
    for (const ProfRec& r : g_recs) {
        if (kind >= 0 && r.kind != kind) continue;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return cuda_fail(e, "profiler event sync");
        float x = 0.f;
        e = cudaEventElapsedTime(&x, r.a, r.b);
        if (e != cudaSuccess) return cuda_fail(e, "profiler elapsed time");
        t += x;
        f += r.flops;
        n++;
    }
    *ms = t;
    *flops = f;
    *launches = n;
    return CAFFE_OK;
}

caffe_status caffe_set_tuning(int32_t key, int32_t value) {
    if (key == CAFFE_TUNE_HALO_EPI_GROUPS) {
        if (value != 0 && (value < 2 || value > 4)) return fail(CAFFE_E_PARAM, "halo epilogue groups must be 0 (auto), 2, 3 or 4");
        g_halo_epi_groups = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_LRN_BWD_C16) {
        cb::g_lrn_bwd_c16 = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_POOL_LRN_C16) {
        cb::g_pool_lrn_c16 = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_IP_FWD_SMALL_BN) {
        if (value != 0 && value != 64 && value != 128) return fail(CAFFE_E_PARAM, "small-output inner-product N tile must be 0, 64 or 128");
        g_ip_fwd_small_bn = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_PDL) {
        cb::g_pdl = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_BIAS_SPLIT_ROWS) {
        if (value < 8 || value > 1024) return fail(CAFFE_E_PARAM, "bias split rows must be 8 .. 1024");
        cb::g_bias_split_rows = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_BIAS_ROWS) {
        cb::g_bias_rows = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_ROWS_CB) {
        cb::g_rows_cb = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_I8_ROWS) {
        if (value < 0 || value > 2) return fail(CAFFE_E_PARAM, "I8 pack form must be 0, 1 or 2");
        cb::g_i8_rows = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_IP_MAX_SPLITS) {
        if (value < 0 || value > 64) return fail(CAFFE_E_PARAM, "inner-product split cap must be 0 (none) .. 64");
        g_ip_max_splits = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_MERGE) {
        g_halo_merge = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_WGRAD_BN) {
        if (value < 0 || value > 256 || (value % 16 && value != 1 && value != 2))
            return fail(CAFFE_E_PARAM, "weight-gradient N tile must be 0 (auto), 1 (widest <= 192) or a multiple of 16 <= 256");
        g_wgrad_bn = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_JN) {
        g_halo_jn = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_BTAPS) {
        if (value < 0 || value > 8) return fail(CAFFE_E_PARAM, "halo B taps per stage must be 0 (auto) .. 8");
        g_halo_btaps = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_WGRAD_REDUCE_WIDE) {
        cb::g_wgrad_reduce_wide = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_COALESCE) {
        cb::g_halo_coal = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_FUSED_POOL_ROWS) {
        if (value < 0 || value > 64) return fail(CAFFE_E_PARAM, "fused pool rows must be 0 (auto) .. 64");
        cb::g_fused_rb = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_MAX_CTAS) {
        if (value < 0) return fail(CAFFE_E_PARAM, "max CTAs must be >= 0 (0 = one per SM)");
        g_max_ctas = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_CTA_PAIR) {
        if (value < 0 || value > 2) return fail(CAFFE_E_PARAM, "CTA-pair mode must be 0 (auto), 1 or 2");
        g_force_cg = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_MMA_SPIN) {
        g_mma_spin = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_TMA_STORE) {
        g_tma_store = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_SGD_BLOCKS_PER_SM) {
        if (value < 0 || value > 8) return fail(CAFFE_E_PARAM, "SGD blocks per SM must be 0 (default 4) .. 8");
        g_sgd_blocks_per_sm = value == 0 ? 4 : value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_SGD_THREADS) {
        if (value != 0 && value != 64 && value != 128 && value != 256)
            return fail(CAFFE_E_PARAM, "SGD threads per block must be 0 (default 256), 64, 128 or 256");
        cb::g_sgd_threads = value == 0 ? 256 : value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_STACKED) {
        if (value < 0 || value > 4)
            return fail(CAFFE_E_PARAM, "stacked halo mode must be 0 (off), 1 (auto), 2 (force), 3 (force, 2 accumulators "
                                       "to 256 columns), 4 (force, N tiles split to <= 128 columns)");
        g_halo_stacked = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_WGRAD_REDUCE_ROWS) {
        cb::g_wgrad_reduce_rows = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_TMA_STORE) {
        cb::g_halo_tma_store = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_FAST_EPI) {
        cb::g_halo_fast_epi = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO_KTRIM) {
        g_halo_ktrim = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_WGRAD_REDUCE_SG) {
        if (value < 0) return fail(CAFFE_E_PARAM, "split-group reduction threshold must be >= 0 (0 = default 24)");
        g_wgrad_reduce_sg_min = value == 0 ? 24 : value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_POOL_STRIP_ROWS) {
        if (value < 0 || value > 1024) return fail(CAFFE_E_PARAM, "pool strip rows must be 0 (auto) .. 1024");
        g_pool_strip_rows = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_ROWS_EPILOGUE) {
        g_rows_epi = value ? 1 : 0;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_HALO) {
        if (value < 0 || value > 3) return fail(CAFFE_E_PARAM, "halo mode must be 0 (auto), 1 (off), 2 (force), 3 (force, <=128-row tiles)");
        g_halo = value;
        return CAFFE_OK;
    }
    if (key == CAFFE_TUNE_WGRAD_MACC) {
        if (value < 0 || value > 4) return fail(CAFFE_E_PARAM, "weight-gradient accumulators per unit must be 0 (auto) .. 4");
        g_wgrad_macc = value;
        return CAFFE_OK;
    }
    return fail(CAFFE_E_INVALID, "unknown tuning key %d", key);
}

caffe_status caffe_device_check(void) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) return fail(CAFFE_E_ARCH, "device is sm_%d%d, this library is built for sm_100a", major, minor);
    return CAFFE_OK;
}

caffe_status caffe_conv_output_shape(const caffe_conv_desc* desc, caffe_shape4 bottom, int32_t num_output,
                                     caffe_shape4* top) {
    if (!top) return fail(CAFFE_E_INVALID, "top is NULL");
    Plan p;
    caffe_status st = conv_validate(desc, bottom, num_output, &p);
    if (st) return st;
    *top = caffe_shape4{bottom.n, num_output, p.OH, p.OW};
    return CAFFE_OK;
}

caffe_status caffe_conv_workspace_size(const caffe_conv_desc* desc, caffe_shape4 bottom, caffe_shape4 weight,
                                       int32_t pass, size_t* bytes) {
    if (!bytes) return fail(CAFFE_E_INVALID, "bytes is NULL");
    if (pass < 0 || pass > 2) return fail(CAFFE_E_INVALID, "bad pass %d", pass);
    Plan p;
    caffe_status st = conv_validate(desc, bottom, weight.n, &p);
    if (st) return st;
    *bytes = bottom.n == 0 ? 0 : conv_ws(p, pass, desc->math);
    return CAFFE_OK;
}

static caffe_status conv_common(const caffe_conv_desc* desc, const caffe_blob* bottom_like, const caffe_blob* weight,
                                Plan* p, bool i8_ok = false) {
    caffe_status st;
    if (i8_ok && bottom_like && bottom_like->dtype == CAFFE_I8) {
        // integer image input: channels-last, tensor-core math, packed by caffe_conv_pack_bottom
        caffe_blob tmp = *bottom_like;
        tmp.dtype = CAFFE_BF16;
        if ((st = check_blob(&tmp, "bottom"))) return st;
        if (!nhwc(bottom_like) || desc->math != CAFFE_MATH_BF16)
            return fail(CAFFE_E_DTYPE, "I8 bottom needs channels-last layout and BF16 math");
    } else if ((st = check_blob(bottom_like, "bottom"))) {
        return st;
    }
    if ((st = check_blob(weight, "weight"))) return st;
    if ((st = conv_validate(desc, bottom_like->shape, weight->shape.n, p))) return st;
    if (weight->shape.c != p->Cg || weight->shape.h != p->kh || weight->shape.w != p->kw)
        return fail(CAFFE_E_SHAPE, "weight shape (%d,%d,%d,%d) != (O,C/g,kh,kw) = (%d,%d,%d,%d)", weight->shape.n,
                    weight->shape.c, weight->shape.h, weight->shape.w, p->O, p->Cg, p->kh, p->kw);
    if (desc->math == CAFFE_MATH_TF32 && (bottom_like->dtype == CAFFE_BF16 || weight->dtype == CAFFE_BF16))
        return fail(CAFFE_E_DTYPE, "TF32 math with BF16 storage");
    return CAFFE_OK;
}

caffe_status caffe_conv_pack_bottom(const caffe_conv_desc* desc, const caffe_blob* bottom, const caffe_blob* weight,
                                    void* ws, size_t ws_bytes, caffe_stream_t stream) {
    Plan p;
    caffe_status st = conv_common(desc, bottom, weight, &p, true);
    if (st) return st;
    if (desc->math == CAFFE_MATH_FP32 || p.N == 0) return CAFFE_OK;
    const size_t need = std::max(conv_ws(p, CAFFE_PASS_FORWARD, desc->math),
                                 conv_ws(p, CAFFE_PASS_BACKWARD_WEIGHT, desc->math));
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    Operand A = plan_x(bottom, p);
    if (bottom->dtype == CAFFE_I8) {
        if (!A.packed) A = Operand{nullptr, 0, 0, 0, 0, true, PackGeom{p.N, p.C, p.H, p.W, p.G, p.Cg, p.bh, p.bw, 0, 0,
                                                                          p.H, p.W, round_ch(p.Cge, p.E),
                                                                          p.G * round_ch(p.Cge, p.E)}};
        CK(pack_act_i8(bottom->ptr, ws, A.pg, (cudaStream_t)stream), "pack I8 activations");
        return CAFFE_OK;
    }
    return pack_if(A, bottom, ws, p.E, (cudaStream_t)stream);
}

caffe_status caffe_conv_pack_weights(const caffe_conv_desc* desc, caffe_shape4 bottom, const caffe_blob* weight,
                                     int32_t pass, void* ws, size_t ws_bytes, caffe_stream_t stream) {
    caffe_status st;
    if (!desc) return fail(CAFFE_E_INVALID, "desc is NULL");
    if ((st = check_blob(weight, "weight"))) return st;
    Plan p;
    if ((st = conv_validate(desc, bottom, weight->shape.n, &p))) return st;
    if (weight->shape.c != p.Cg || weight->shape.h != p.kh || weight->shape.w != p.kw)
        return fail(CAFFE_E_SHAPE, "weight shape (%d,%d,%d,%d) != (O,C/g,kh,kw) = (%d,%d,%d,%d)", weight->shape.n,
                    weight->shape.c, weight->shape.h, weight->shape.w, p.O, p.Cg, p.kh, p.kw);
    if (pass != CAFFE_PASS_FORWARD && pass != CAFFE_PASS_BACKWARD_DATA)
        return fail(CAFFE_E_INVALID, "pass must be CAFFE_PASS_FORWARD or CAFFE_PASS_BACKWARD_DATA");
    if (desc->math == CAFFE_MATH_FP32 || p.N == 0) return CAFFE_OK;
    const size_t need = conv_ws(p, pass, desc->math);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    char* w8 = (char*)ws;
    cudaStream_t s = (cudaStream_t)stream;
    if (pass == CAFFE_PASS_FORWARD)
        CK(repack_w_fwd(weight->ptr, isbf(weight), w8 + ws_x_max(p), p.E, wgeom(p), s), "repack weights");
    else
        CK(repack_w_dgrad(weight->ptr, isbf(weight), w8 + ws_dy_max(p), p.E, wgeom(p), p.Cge, s), "repack weights (dgrad)");
    return CAFFE_OK;
}

caffe_status caffe_conv_forward(const caffe_conv_desc* desc, const caffe_blob* bottom, const caffe_blob* weight,
                                const caffe_blob* bias, caffe_blob* top, void* ws, size_t ws_bytes,
                                caffe_stream_t stream) {
    Plan p;
    caffe_status st = conv_common(desc, bottom, weight, &p, desc && (desc->flags & CAFFE_BOTTOM_PREPACKED));
    if (st) return st;
    if ((st = check_blob(top, "top"))) return st;
    if (bias) {
        if ((st = check_blob(bias, "bias"))) return st;
        if (bias->dtype != CAFFE_F32) return fail(CAFFE_E_DTYPE, "bias must be F32");
        if (cnt(bias->shape) != p.O) return fail(CAFFE_E_SHAPE, "bias has %lld elements, num_output %d", cnt(bias->shape), p.O);
    }
    caffe_shape4 want{p.N, p.O, p.OH, p.OW};
    if (!same_shape(top->shape, want))
        return fail(CAFFE_E_SHAPE, "top shape (%d,%d,%d,%d) != (%d,%d,%d,%d)", top->shape.n, top->shape.c, top->shape.h,
                    top->shape.w, want.n, want.c, want.h, want.w);
    if (overlap(top, bottom) || overlap(top, weight) || overlap(top, bias)) return fail(CAFFE_E_ALIAS, "top overlaps an input");
    if (desc->math == CAFFE_MATH_TF32 && top->dtype == CAFFE_BF16) return fail(CAFFE_E_DTYPE, "TF32 math with BF16 storage");
    if (p.N == 0) return CAFFE_OK;
    const size_t need = conv_ws(p, CAFFE_PASS_FORWARD, desc->math);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    const int relu = (desc->flags & CAFFE_FUSE_RELU) ? 1 : 0;
    const float* bptr = bias ? (const float*)bias->ptr : nullptr;
    if (desc->math == CAFFE_MATH_FP32) {
        CK(fp32_conv_fwd(bottom->ptr, isbf(bottom), strides(bottom), weight->ptr, isbf(weight), bptr, top->ptr, isbf(top),
                         strides(top), nhwc(top), relu, cgeom(p), s),
           "conv fwd fp32");
        return CAFFE_OK;
    }
    char* w8 = (char*)ws;
    Operand A = plan_x(bottom, p);
    void* XA = w8;
    void* WB = w8 + ws_x_max(p);
    if (!(desc->flags & CAFFE_BOTTOM_PREPACKED) && (st = pack_if(A, bottom, XA, p.E, s))) return st;
    const void* aptr = A.packed ? XA : A.ptr;
    if (!(desc->flags & CAFFE_WEIGHTS_PREPACKED)) CK(repack_w_fwd(weight->ptr, isbf(weight), WB, p.E, wgeom(p), s), "repack weights");
    TcLaunch L;
    memset(&L, 0, sizeof L);
    const HaloGeom hg{A.H, A.W, p.OH, p.OW, p.khp, p.kwp, p.php, p.pwp};
    if (halo_applies(p.E, hg) || stacked_applies(p.E, hg, halo_bn(p.Og, hg))) {
        TcArgs& a = L.args;
        a.BN = halo_bn(p.Og, hg); a.N = p.Og;
        a.n_tiles = (int)cdiv(p.Og, a.BN); a.groups = p.G;
        a.a_cblocks = p.Cgp / p.CH; a.a_cpg = A.cpg; a.b_row_g = p.Og;
        set_out(a, top);
        a.col_g = p.Og; a.bias = bptr; a.relu = relu; a.beta = 0.f;
        a.k_last = g_halo_ktrim ? (int)cdiv(p.Cge - p.CH * (a.a_cblocks - 1), 16) : 0;
        if (!halo_setup(L, hg, aptr, A.Ctot, p.N)) return fail(CAFFE_E_CUDA, "halo tile setup failed (activation)");
        if (!encode_tiled_2d(&L.mapB, p.E, WB, (uint64_t)p.taps * p.Cgp, (uint64_t)p.O, (uint64_t)p.taps * p.Cgp * p.E,
                             p.CH, a.BN / L.cg))
            return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (weights)");
        return run_tc(L, s, conv_flops(p), 0);
    }
    L.esz = p.E; L.amode = A_IM2COL_K; L.bmode = B_TILED_K; L.epi = EPI_STRIDED;
    if (!encode_im2col_4d(&L.mapA, p.E, aptr, A.Ctot, A.W, A.H, p.N, p.pwp, p.php, p.pwp - (p.kwp - 1),
                          p.php - (p.khp - 1), p.CH, 128))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeIm2col failed (activation)");
    TcArgs& a = L.args;
    a.BN = choose_bn(p.Og);
    a.M = p.N * p.OH * p.OW; a.N = p.Og;
    a.n_tiles = (int)cdiv(p.Og, a.BN); a.groups = p.G; a.splits = 1;
    L.cg = pick_cg(a.M, a.n_tiles * p.G, p.E);
    a.m_tiles = (int)cdiv(a.M, 128 * L.cg);
    if (!encode_tiled_2d(&L.mapB, p.E, WB, (uint64_t)p.taps * p.Cgp, (uint64_t)p.O, (uint64_t)p.taps * p.Cgp * p.E,
                         p.CH, a.BN / L.cg))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (weights)");
    a.kblocks = p.taps * (p.Cgp / p.CH); a.kb_per_split = a.kblocks;
    a.a_P = p.OH * p.OW; a.a_OW = p.OW; a.a_pad_h = p.php; a.a_pad_w = p.pwp; a.a_kw = p.kwp;
    a.a_cblocks = p.Cgp / p.CH; a.a_cpg = A.cpg; a.b_row_g = p.Og;
    set_out(a, top);
    a.col_g = p.Og; a.bias = bptr; a.relu = relu; a.beta = 0.f;
    finish_args(a, a.BN / L.cg * 128);
    if (nhwc(top))
        enable_tma_store(L, top->ptr, isbf(top) ? 2 : 4, p.O, (long long)p.N * p.OH * p.OW, p.O,
                         p.G == 1 || p.Og % a.BN == 0);
    return run_tc(L, s, conv_flops(p), 0);
}

static caffe_status conv_bwd_data(const caffe_conv_desc* desc, const caffe_blob* top_diff, const caffe_blob* weight,
                                  const caffe_blob* relu_top, caffe_blob* bottom_diff, float beta, void* ws,
                                  size_t ws_bytes, caffe_stream_t stream);

caffe_status caffe_conv_backward_data(const caffe_conv_desc* desc, const caffe_blob* top_diff, const caffe_blob* weight,
                                      caffe_blob* bottom_diff, float beta, void* ws, size_t ws_bytes,
                                      caffe_stream_t stream) {
    return conv_bwd_data(desc, top_diff, weight, nullptr, bottom_diff, beta, ws, ws_bytes, stream);
}

caffe_status caffe_conv_backward_data_relu(const caffe_conv_desc* desc, const caffe_blob* top_diff,
                                           const caffe_blob* weight, const caffe_blob* relu_top, caffe_blob* bottom_diff,
                                           void* ws, size_t ws_bytes, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(relu_top, "relu_top"))) return st;
    if ((st = check_blob(bottom_diff, "bottom_diff"))) return st;
    if (!same_shape(relu_top->shape, bottom_diff->shape))
        return fail(CAFFE_E_SHAPE, "relu_top shape (%d,%d,%d,%d) != bottom_diff shape (%d,%d,%d,%d)", relu_top->shape.n,
                    relu_top->shape.c, relu_top->shape.h, relu_top->shape.w, bottom_diff->shape.n, bottom_diff->shape.c,
                    bottom_diff->shape.h, bottom_diff->shape.w);
    if (nhwc(relu_top) != nhwc(bottom_diff)) return fail(CAFFE_E_INVALID, "relu_top and bottom_diff layouts differ");
    if (overlap(bottom_diff, relu_top)) return fail(CAFFE_E_ALIAS, "bottom_diff overlaps relu_top");
    return conv_bwd_data(desc, top_diff, weight, relu_top, bottom_diff, 0.f, ws, ws_bytes, stream);
}

static caffe_status conv_bwd_data(const caffe_conv_desc* desc, const caffe_blob* top_diff, const caffe_blob* weight,
                                  const caffe_blob* relu_top, caffe_blob* bottom_diff, float beta, void* ws,
                                  size_t ws_bytes, caffe_stream_t stream) {
    Plan p;
    caffe_status st;
    if ((st = check_blob(bottom_diff, "bottom_diff"))) return st;
    if ((st = conv_common(desc, bottom_diff, weight, &p))) return st;
    if ((st = check_blob(top_diff, "top_diff"))) return st;
    caffe_shape4 want{p.N, p.O, p.OH, p.OW};
    if (!same_shape(top_diff->shape, want))
        return fail(CAFFE_E_SHAPE, "top_diff shape (%d,%d,%d,%d) != (%d,%d,%d,%d)", top_diff->shape.n, top_diff->shape.c,
                    top_diff->shape.h, top_diff->shape.w, want.n, want.c, want.h, want.w);
    if (overlap(bottom_diff, top_diff) || overlap(bottom_diff, weight)) return fail(CAFFE_E_ALIAS, "bottom_diff overlaps an input");
    if (desc->math == CAFFE_MATH_TF32 && top_diff->dtype == CAFFE_BF16) return fail(CAFFE_E_DTYPE, "TF32 math with BF16 storage");
    if (p.N == 0) return CAFFE_OK;
    const size_t need = conv_ws(p, CAFFE_PASS_BACKWARD_DATA, desc->math);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    // ReLU backward by a separate in-place pass where the epilogue does not take it (beta is 0 here)
    const long long bcount = (long long)p.N * p.C * p.H * p.W;
    auto relu_after = [&]() -> caffe_status {
        if (relu_top)
            CK(relu_bwd(relu_top->ptr, bottom_diff->ptr, bottom_diff->ptr, isbf(relu_top), isbf(bottom_diff), (int)bcount,
                        s),
               "relu backward");
        return CAFFE_OK;
    };
    if (desc->math == CAFFE_MATH_FP32) {
        CK(fp32_conv_dgrad(top_diff->ptr, isbf(top_diff), strides(top_diff), weight->ptr, isbf(weight), bottom_diff->ptr,
                           isbf(bottom_diff), nhwc(bottom_diff), beta, cgeom(p), s),
           "conv dgrad fp32");
        return relu_after();
    }
    char* w8 = (char*)ws;
    Operand A = plan_dy(top_diff, p);
    void* DYA = w8;
    void* WD = w8 + ws_dy_max(p);
    float* T = (float*)(w8 + ws_dy_max(p) + ws_wd(p));
    if ((st = pack_if(A, top_diff, DYA, p.E, s))) return st;
    const void* aptr = A.packed ? DYA : A.ptr;
    if (!(desc->flags & CAFFE_WEIGHTS_PREPACKED))
        CK(repack_w_dgrad(weight->ptr, isbf(weight), WD, p.E, wgeom(p), p.Cge, s), "repack weights (dgrad)");
    const int Hd = p.s2d ? p.Hp : p.H, Wd = p.s2d ? p.Wp : p.W;
    const int lo_h = p.khp - 1 - p.php, lo_w = p.kwp - 1 - p.pwp;
    TcLaunch L;
    memset(&L, 0, sizeof L);
    const HaloGeom hg{p.OH, p.OW, Hd, Wd, p.khp, p.kwp, lo_h, lo_w};
    if (!p.s2d && (halo_applies(p.E, hg) || stacked_applies(p.E, hg, halo_bn(p.Cge, hg)))) {
        TcArgs& a = L.args;
        a.BN = halo_bn(p.Cge, hg); a.N = p.Cge;
        a.n_tiles = (int)cdiv(p.Cge, a.BN); a.groups = p.G;
        a.a_cblocks = p.Ogp / p.CH; a.a_cpg = A.cpg; a.b_row_g = p.Cge;
        set_out(a, bottom_diff);
        a.col_g = p.Cg; a.beta = beta;
        if (relu_top) { a.relu_top = relu_top->ptr; a.relu_top_bf16 = isbf(relu_top); }
        a.k_last = g_halo_ktrim ? (int)cdiv(p.Og - p.CH * (a.a_cblocks - 1), 16) : 0;
        if (!halo_setup(L, hg, aptr, A.Ctot, p.N)) return fail(CAFFE_E_CUDA, "halo tile setup failed (top_diff)");
        if (jn_setup(L, p, bottom_diff, relu_top, beta, WD)) return run_tc(L, s, conv_flops(p), 0);
        if (!encode_tiled_2d(&L.mapB, p.E, WD, (uint64_t)p.taps * p.Ogp, (uint64_t)p.G * p.Cge,
                             (uint64_t)p.taps * p.Ogp * p.E, p.CH, a.BN / L.cg))
            return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (dgrad weights)");
        return run_tc(L, s, conv_flops(p), 0);
    }
    L.esz = p.E; L.amode = A_IM2COL_K; L.bmode = B_TILED_K; L.epi = EPI_STRIDED;
    if (!encode_im2col_4d(&L.mapA, p.E, aptr, A.Ctot, p.OW, p.OH, p.N, lo_w, lo_h, lo_w - (p.kwp - 1),
                          lo_h - (p.khp - 1), p.CH, 128))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeIm2col failed (top_diff)");
    TcArgs& a = L.args;
    a.BN = choose_bn(p.Cge);
    a.M = p.N * Hd * Wd; a.N = p.Cge;
    a.n_tiles = (int)cdiv(p.Cge, a.BN); a.groups = p.G; a.splits = 1;
    L.cg = pick_cg(a.M, a.n_tiles * p.G, p.E);
    a.m_tiles = (int)cdiv(a.M, 128 * L.cg);
    if (!encode_tiled_2d(&L.mapB, p.E, WD, (uint64_t)p.taps * p.Ogp, (uint64_t)p.G * p.Cge,
                         (uint64_t)p.taps * p.Ogp * p.E, p.CH, a.BN / L.cg))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (dgrad weights)");
    a.kblocks = p.taps * (p.Ogp / p.CH); a.kb_per_split = a.kblocks;
    a.a_P = Hd * Wd; a.a_OW = Wd; a.a_pad_h = lo_h; a.a_pad_w = lo_w; a.a_kw = p.kwp;
    a.a_cblocks = p.Ogp / p.CH; a.a_cpg = A.cpg; a.b_row_g = p.Cge;
    PackGeom tg{p.N, p.C, p.H, p.W, p.G, p.Cg, p.bh, p.bw, p.ph, p.pw, p.Hp, p.Wp, p.Cge, p.G * p.Cge};
    if (!p.s2d) {
        set_out(a, bottom_diff);
        a.col_g = p.Cg; a.beta = beta;
        if (relu_top) { a.relu_top = relu_top->ptr; a.relu_top_bf16 = isbf(relu_top); }
    } else {
        a.out = T; a.out_bf16 = 0; a.P = p.Hp * p.Wp;
        a.s_n = (long long)p.Hp * p.Wp * tg.Ctot; a.s_c = 1; a.s_p = tg.Ctot;
        a.col_g = p.Cge; a.beta = 0.f;
    }
    finish_args(a, a.BN / L.cg * 128);
    // the TMA-store epilogue takes the ReLU mask for BF16 output and reference in whole 64-column chunks
    const bool tma_ok = !relu_top || (isbf(bottom_diff) && isbf(relu_top) && p.Cge % 64 == 0);
    if (!p.s2d && nhwc(bottom_diff) && tma_ok)
        enable_tma_store(L, bottom_diff->ptr, isbf(bottom_diff) ? 2 : 4, p.C, (long long)p.N * p.H * p.W, p.C,
                         p.G == 1 || p.Cg % a.BN == 0);
    if ((st = run_tc(L, s, conv_flops(p), 0))) return st;
    if (p.s2d) {
        CK(unpack_s2d_grad(T, bottom_diff->ptr, isbf(bottom_diff), nhwc(bottom_diff), beta, tg, s), "unpack s2d gradient");
        return relu_after();
    }
    return CAFFE_OK;
}

caffe_status caffe_conv_backward_weight(const caffe_conv_desc* desc, const caffe_blob* bottom,
                                        const caffe_blob* top_diff, caffe_blob* weight_diff, caffe_blob* bias_diff,
                                        float beta, void* ws, size_t ws_bytes, caffe_stream_t stream) {
    Plan p;
    caffe_status st;
    if ((st = conv_common(desc, bottom, weight_diff, &p, desc && (desc->flags & CAFFE_BOTTOM_PREPACKED)))) return st;
    if ((st = check_blob(top_diff, "top_diff"))) return st;
    if (weight_diff->dtype != CAFFE_F32) return fail(CAFFE_E_DTYPE, "weight_diff must be F32");
    caffe_shape4 want{p.N, p.O, p.OH, p.OW};
    if (!same_shape(top_diff->shape, want))
        return fail(CAFFE_E_SHAPE, "top_diff shape (%d,%d,%d,%d) != (%d,%d,%d,%d)", top_diff->shape.n, top_diff->shape.c,
                    top_diff->shape.h, top_diff->shape.w, want.n, want.c, want.h, want.w);
    if (bias_diff) {
        if ((st = check_blob(bias_diff, "bias_diff"))) return st;
        if (bias_diff->dtype != CAFFE_F32) return fail(CAFFE_E_DTYPE, "bias_diff must be F32");
        if (cnt(bias_diff->shape) != p.O) return fail(CAFFE_E_SHAPE, "bias_diff has %lld elements, num_output %d", cnt(bias_diff->shape), p.O);
    }
    if (overlap(weight_diff, bottom) || overlap(weight_diff, top_diff) || overlap(bias_diff, bottom) ||
        overlap(bias_diff, top_diff) || overlap(bias_diff, weight_diff))
        return fail(CAFFE_E_ALIAS, "weight_diff/bias_diff overlaps an input");
    if (desc->math == CAFFE_MATH_TF32 && top_diff->dtype == CAFFE_BF16) return fail(CAFFE_E_DTYPE, "TF32 math with BF16 storage");
    if (p.N == 0) return CAFFE_OK;
    const size_t need = conv_ws(p, CAFFE_PASS_BACKWARD_WEIGHT, desc->math);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    char* w8 = (char*)ws;
    // FP32 math: CUDA-core FP32 FMA (blocked reduction, R13).  TF32 runs on the tensor cores below
    // (tcgen05.mma kind::tf32 with MN-major operands: both packed TF32-RN, as in the other passes).
    if (desc->math == CAFFE_MATH_FP32) {
        if (bias_diff)
            CK(bias_grad(top_diff->ptr, isbf(top_diff), nhwc(top_diff), (float*)bias_diff->ptr, beta, p.N, p.O,
                         p.OH * p.OW, (float*)w8, s),
               "bias grad");
        CK(fp32_conv_wgrad(bottom->ptr, isbf(bottom), strides(bottom), top_diff->ptr, isbf(top_diff), strides(top_diff),
                           (float*)weight_diff->ptr, beta, cgeom(p), s, 0),
           "conv wgrad fp32");
        return CAFFE_OK;
    }
    Operand A = plan_x(bottom, p);
    Operand B = plan_dy(top_diff, p);
    void* XA = w8;
    void* DYA = w8 + ws_x_max(p);
    float* PART = (float*)(w8 + ws_x_max(p) + ws_dy_max(p));
    float* BPART = (float*)(w8 + ws_x_max(p) + ws_dy_max(p) + ws_partial(p));
    const WgHalo hw = wgrad_halo_plan(p);
    // bias gradient inside the halo weight gradient (ones chunk) when dY feeds the MMA unmodified
    // (bf16, read in place) and the tap count leaves a spare chunk; else a separate reduction
    const bool bias_mma = bias_diff && hw.use && !B.packed && isbf(top_diff) && (p.taps & 1) == 1;
    if (bias_diff && !bias_mma)
        CK(bias_grad(top_diff->ptr, isbf(top_diff), nhwc(top_diff), (float*)bias_diff->ptr, beta, p.N, p.O,
                     p.OH * p.OW, BPART, s),
           "bias grad");
    if (!(desc->flags & CAFFE_BOTTOM_PREPACKED) && (st = pack_if(A, bottom, XA, p.E, s))) return st;
    if ((st = pack_if(B, top_diff, DYA, p.E, s))) return st;
    const void* aptr = A.packed ? XA : A.ptr;
    const void* bptr = B.packed ? DYA : B.ptr;
    if (hw.use) {
        TcLaunch L;
        memset(&L, 0, sizeof L);
        L.esz = 2; L.amode = A_HALO_MN; L.bmode = B_TILED_MN; L.epi = EPI_PARTIAL; L.cg = 1;
        if (!encode_tiled_4d(&L.mapA, 2, aptr, A.Ctot, A.W, A.H, p.N, 64, (uint32_t)hw.Wt, (uint32_t)hw.rows) ||
            !encode_tiled_4d(&L.mapB, 2, bptr, B.Ctot, p.OW, p.OH, p.N, 64, (uint32_t)hw.Wt, (uint32_t)hw.TH))
            return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (halo weight gradient)");
        TcArgs& a = L.args;
        a.BN = hw.BN; a.N = p.Og; a.n_tiles = hw.n_tiles; a.groups = p.G;
        a.splits = hw.splits; a.kb_per_split = hw.kb_per; a.total_tiles = hw.total; a.tiles_per_img = hw.tpi;
        a.halo_wt = hw.Wt; a.halo_th = hw.TH; a.halo_rows = hw.rows; a.halo_kh = p.khp; a.a_kw = p.kwp;
        a.a_pad_h = p.php; a.a_pad_w = p.pwp; a.a_cpg = A.cpg; a.b_col_g = B.cpg;
        a.b_nchunks = hw.nch; a.b_stage_bytes = hw.nch * hw.bchunk; a.halo_slot = hw.slot; a.stages = hw.stages;
        a.acc_stride = hw.acc_stride; a.macc = hw.macc; a.m_tiles_real = hw.pairs; a.m_tiles = hw.mgroups;
        a.a_cblocks = hw.cblocks; a.halo_ksteps = hw.ksteps; a.bias_mma = bias_mma ? 1 : 0;
        a.tmem_cols = 512; a.partial = PART;
        a.units = p.G * hw.n_tiles * hw.mgroups * hw.cblocks * hw.splits;
        if ((st = run_tc(L, s, conv_flops(p), 0))) return st;
        CK(wgrad_reduce(PART, (float*)weight_diff->ptr, beta, wgeom(p), hw.cblocks * hw.pairs, hw.n_tiles, hw.splits,
                        hw.BN, 64, hw.cblocks, s, 1, bias_mma ? (float*)bias_diff->ptr : nullptr),
           "wgrad reduce");
        return CAFFE_OK;
    }
    WgradSplit w = wgrad_split(p);
    TcLaunch L;
    memset(&L, 0, sizeof L);
    L.esz = p.E; L.amode = A_IM2COL_MN; L.bmode = B_TILED_MN; L.epi = EPI_PARTIAL;
    if (!encode_im2col_4d(&L.mapA, p.E, aptr, A.Ctot, A.W, A.H, p.N, p.pwp, p.php, p.pwp - (p.kwp - 1),
                          p.php - (p.khp - 1), p.CH, p.CH, p.E == 4))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeIm2col failed (wgrad activation)");
    if (!encode_tiled_2d(&L.mapB, p.E, bptr, (uint64_t)B.Ctot, (uint64_t)p.N * p.OH * p.OW, (uint64_t)B.Ctot * p.E,
                         p.CH, p.CH, p.E == 4))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (wgrad top_diff)");
    TcArgs& a = L.args;
    a.BN = w.BN; a.M = 128 * w.m_tiles; a.N = p.Og;
    a.m_tiles = w.m_groups; a.m_tiles_real = w.m_tiles; a.macc = w.macc;
    a.n_tiles = w.n_tiles; a.groups = p.G; a.splits = w.splits;
    a.kblocks = w.kblocks; a.kb_per_split = w.kb_per;
    a.a_P = p.OH * p.OW; a.a_OW = p.OW; a.a_pad_h = p.php; a.a_pad_w = p.pwp; a.a_kw = p.kwp;
    a.a_cblocks = p.Cgp / p.CH; a.a_cpg = A.cpg; a.a_nchunks_total = p.taps * (p.Cgp / p.CH);
    a.b_col_g = B.cpg; a.b_nchunks = (int)cdiv(w.BN, p.CH);
    a.partial = PART;
    finish_args(a, a.b_nchunks * p.CH * 128);
    if ((st = run_tc(L, s, conv_flops(p), 0))) return st;
    CK(wgrad_reduce(PART, (float*)weight_diff->ptr, beta, wgeom(p), w.m_tiles, w.n_tiles, w.splits, w.BN, p.CH,
                    p.Cgp / p.CH, s),
       "wgrad reduce");
    return CAFFE_OK;
}

// ------------------------------------------------------------------ ReLU
caffe_status caffe_relu_forward(const caffe_blob* bottom, caffe_blob* top, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom, "bottom")) || (st = check_blob(top, "top"))) return st;
    if (!same_shape(bottom->shape, top->shape) || bottom->dtype != top->dtype || bottom->layout != top->layout)
        return fail(CAFFE_E_SHAPE, "top must match bottom in shape, dtype and layout");
    if (bottom->ptr != top->ptr && overlap(bottom, top)) return fail(CAFFE_E_ALIAS, "partial overlap of top and bottom");
    if (cnt(bottom->shape) == 0) return CAFFE_OK;
    if (!aligned16(bottom->ptr) || !aligned16(top->ptr)) return fail(CAFFE_E_ALIGN, "ReLU buffers must be 16-byte aligned");
    CK(relu_fwd(bottom->ptr, top->ptr, isbf(bottom), (int)cnt(bottom->shape), (cudaStream_t)stream), "relu fwd");
    return CAFFE_OK;
}

caffe_status caffe_relu_backward(const caffe_blob* x, const caffe_blob* top_diff, caffe_blob* bottom_diff,
                                 caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(x, "bottom_or_top")) || (st = check_blob(top_diff, "top_diff")) ||
        (st = check_blob(bottom_diff, "bottom_diff")))
        return st;
    if (!same_shape(x->shape, top_diff->shape) || !same_shape(x->shape, bottom_diff->shape) ||
        top_diff->dtype != bottom_diff->dtype || x->layout != top_diff->layout || x->layout != bottom_diff->layout)
        return fail(CAFFE_E_SHAPE, "ReLU backward blobs must share shape and layout (and diff dtype)");
    if ((bottom_diff->ptr != top_diff->ptr && overlap(bottom_diff, top_diff)) || overlap(bottom_diff, x))
        return fail(CAFFE_E_ALIAS, "bottom_diff overlaps an input");
    if (cnt(x->shape) == 0) return CAFFE_OK;
    CK(relu_bwd(x->ptr, top_diff->ptr, bottom_diff->ptr, isbf(x), isbf(top_diff), (int)cnt(x->shape), (cudaStream_t)stream),
       "relu bwd");
    return CAFFE_OK;
}

// ------------------------------------------------------------------ pooling
static caffe_status pool_validate(const caffe_pool_desc* d, caffe_shape4 b, PoolGeom* g) {
    if (!d) return fail(CAFFE_E_INVALID, "desc is NULL");
    if (d->method != CAFFE_POOL_MAX && d->method != CAFFE_POOL_AVE) return fail(CAFFE_E_INVALID, "bad pool method %d", d->method);
    if (d->kernel_h < 1 || d->kernel_w < 1) return fail(CAFFE_E_PARAM, "zero-sized pooling window (S:164)");
    if (d->stride_h < 1 || d->stride_w < 1 || d->pad_h < 0 || d->pad_w < 0)
        return fail(CAFFE_E_PARAM, "bad pool stride/pad");
    if (d->pad_h >= d->kernel_h || d->pad_w >= d->kernel_w) return fail(CAFFE_E_PARAM, "pad must be smaller than the window");
    if (d->kernel_h > b.h + 2 * d->pad_h || d->kernel_w > b.w + 2 * d->pad_w)
        return fail(CAFFE_E_PARAM, "pool window larger than padded input");
    auto od = [](int in, int k, int s, int p) {
        int o = (in + 2 * p - k + s - 1) / s + 1;
        if ((o - 1) * s >= in + p) o -= 1;
        return o;
    };
    *g = PoolGeom{b.n, b.c, b.h, b.w, d->kernel_h, d->kernel_w, d->stride_h, d->stride_w, d->pad_h, d->pad_w,
                  od(b.h, d->kernel_h, d->stride_h, d->pad_h), od(b.w, d->kernel_w, d->stride_w, d->pad_w)};
    return CAFFE_OK;
}

caffe_status caffe_pool_output_shape(const caffe_pool_desc* desc, caffe_shape4 bottom, caffe_shape4* top) {
    if (!top) return fail(CAFFE_E_INVALID, "top is NULL");
    PoolGeom g;
    caffe_status st = pool_validate(desc, bottom, &g);
    if (st) return st;
    *top = caffe_shape4{bottom.n, bottom.c, g.OH, g.OW};
    return CAFFE_OK;
}

caffe_status caffe_pool_forward(const caffe_pool_desc* desc, const caffe_blob* bottom, caffe_blob* top, caffe_blob* mask,
                                caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom, "bottom")) || (st = check_blob(top, "top"))) return st;
    PoolGeom g;
    if ((st = pool_validate(desc, bottom->shape, &g))) return st;
    caffe_shape4 want{g.N, g.C, g.OH, g.OW};
    if (!same_shape(top->shape, want) || top->dtype != bottom->dtype)
        return fail(CAFFE_E_SHAPE, "top shape/dtype mismatch (want %d,%d,%d,%d)", want.n, want.c, want.h, want.w);
    if (mask) {
        if ((st = check_blob(mask, "mask", false))) return st;
        if (!same_shape(mask->shape, want) || mask->layout != top->layout)
            return fail(CAFFE_E_SHAPE, "mask shape/layout must equal top's");
        if (desc->method != CAFFE_POOL_MAX) return fail(CAFFE_E_INVALID, "mask is only produced by MAX pooling");
        if (mask->dtype == CAFFE_U8 && g.kh * g.kw > 255)
            return fail(CAFFE_E_PARAM, "a U8 (window-local) mask needs kernel_h*kernel_w <= 255");
    }
    if (overlap(top, bottom) || overlap(mask, bottom) || overlap(mask, top)) return fail(CAFFE_E_ALIAS, "pool outputs overlap");
    if (g.N == 0) return CAFFE_OK;
    if (desc->method == CAFFE_POOL_MAX)
        CK(maxpool_fwd(bottom->ptr, strides(bottom), top->ptr, nhwc(top), mask ? mask->ptr : nullptr,
                       mask ? (mask->dtype == CAFFE_U8) : 0,
                       isbf(bottom), g, (cudaStream_t)stream),
           "maxpool fwd");
    else
        CK(avepool_fwd(bottom->ptr, strides(bottom), top->ptr, nhwc(top), isbf(bottom), g, (cudaStream_t)stream),
           "avepool fwd");
    return CAFFE_OK;
}

static caffe_status pool_backward_impl(const caffe_pool_desc* desc, const caffe_blob* top, const caffe_blob* top_diff,
                                       const caffe_blob* mask, caffe_blob* bottom_diff, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(top_diff, "top_diff")) || (st = check_blob(bottom_diff, "bottom_diff"))) return st;
    PoolGeom g;
    if ((st = pool_validate(desc, bottom_diff->shape, &g))) return st;
    caffe_shape4 want{g.N, g.C, g.OH, g.OW};
    if (!same_shape(top_diff->shape, want) || top_diff->dtype != bottom_diff->dtype)
        return fail(CAFFE_E_SHAPE, "top_diff shape/dtype mismatch");
    if (desc->method == CAFFE_POOL_MAX) {
        if (!mask) return fail(CAFFE_E_INVALID, "MAX pool backward needs the argmax mask (S:173)");
        if ((st = check_blob(mask, "mask", false))) return st;
        if (!same_shape(mask->shape, want) || mask->layout != top_diff->layout)
            return fail(CAFFE_E_SHAPE, "mask shape/layout must equal top_diff's");
        if (mask->dtype == CAFFE_U8 && g.kh * g.kw > 255)
            return fail(CAFFE_E_PARAM, "a U8 (window-local) mask needs kernel_h*kernel_w <= 255");
    }
    if (top) {
        if (desc->method != CAFFE_POOL_MAX) return fail(CAFFE_E_INVALID, "the ReLU-fused backward needs MAX pooling");
        if ((st = check_blob(top, "top"))) return st;
        if (!same_shape(top->shape, want) || top->dtype != top_diff->dtype || top->layout != top_diff->layout)
            return fail(CAFFE_E_SHAPE, "top must match top_diff (shape, dtype, layout)");
        if (overlap(bottom_diff, top)) return fail(CAFFE_E_ALIAS, "bottom_diff overlaps top");
    }
    if (overlap(bottom_diff, top_diff) || overlap(bottom_diff, mask)) return fail(CAFFE_E_ALIAS, "bottom_diff overlaps an input");
    if (g.N == 0) return CAFFE_OK;
    if (desc->method == CAFFE_POOL_MAX)
        CK(maxpool_bwd(top_diff->ptr, mask->ptr, mask->dtype == CAFFE_U8, top ? top->ptr : nullptr, strides(top_diff),
                       bottom_diff->ptr, nhwc(bottom_diff), isbf(top_diff), g, (cudaStream_t)stream),
           "maxpool bwd");
    else
        CK(avepool_bwd(top_diff->ptr, strides(top_diff), bottom_diff->ptr, nhwc(bottom_diff), isbf(top_diff), g,
                       (cudaStream_t)stream),
           "avepool bwd");
    return CAFFE_OK;
}

caffe_status caffe_pool_backward(const caffe_pool_desc* desc, const caffe_blob* top_diff, const caffe_blob* mask,
                                 caffe_blob* bottom_diff, caffe_stream_t stream) {
    return pool_backward_impl(desc, nullptr, top_diff, mask, bottom_diff, stream);
}

caffe_status caffe_pool_relu_backward(const caffe_pool_desc* desc, const caffe_blob* top, const caffe_blob* top_diff,
                                      const caffe_blob* mask, caffe_blob* bottom_diff, caffe_stream_t stream) {
    if (!top) return fail(CAFFE_E_INVALID, "top is NULL");
    return pool_backward_impl(desc, top, top_diff, mask, bottom_diff, stream);
}

// ------------------------------------------------------------------ LRN
static caffe_status lrn_validate(const caffe_lrn_desc* d) {
    if (!d) return fail(CAFFE_E_INVALID, "desc is NULL");
    if (d->local_size < 1 || d->local_size % 2 == 0) return fail(CAFFE_E_PARAM, "LRN local_size %d must be odd (S:216)", d->local_size);
    if (!(d->k > 0.f) || !(d->beta > 0.f) || d->alpha < 0.f) return fail(CAFFE_E_PARAM, "LRN needs k > 0, beta > 0, alpha >= 0");
    return CAFFE_OK;
}

caffe_status caffe_lrn_forward(const caffe_lrn_desc* desc, const caffe_blob* bottom, caffe_blob* top, caffe_blob* scale,
                               caffe_stream_t stream) {
    caffe_status st;
    if ((st = lrn_validate(desc)) || (st = check_blob(bottom, "bottom")) || (st = check_blob(top, "top"))) return st;
    if (!same_shape(bottom->shape, top->shape) || bottom->dtype != top->dtype || bottom->layout != top->layout)
        return fail(CAFFE_E_SHAPE, "top must match bottom (shape, dtype, layout)");
    if (scale) {
        if ((st = check_blob(scale, "scale"))) return st;
        if (scale->dtype != CAFFE_F32 || !same_shape(scale->shape, bottom->shape) || scale->layout != bottom->layout)
            return fail(CAFFE_E_SHAPE, "scale must be F32 with bottom's shape and layout");
    }
    if (overlap(top, bottom) || overlap(scale, bottom) || overlap(scale, top)) return fail(CAFFE_E_ALIAS, "LRN outputs overlap");
    if (bottom->shape.n == 0) return CAFFE_OK;
    const caffe_shape4& s = bottom->shape;
    CK(lrn_fwd(bottom->ptr, top->ptr, scale ? (float*)scale->ptr : nullptr, isbf(bottom), nhwc(bottom), s.n, s.c, s.h, s.w,
               desc->local_size, desc->alpha, desc->beta, desc->k, (cudaStream_t)stream),
       "lrn fwd");
    return CAFFE_OK;
}

caffe_status caffe_lrn_backward(const caffe_lrn_desc* desc, const caffe_blob* bottom, const caffe_blob* top,
                                const caffe_blob* top_diff, const caffe_blob* scale, caffe_blob* bottom_diff,
                                caffe_stream_t stream) {
    caffe_status st;
    if ((st = lrn_validate(desc)) || (st = check_blob(bottom, "bottom")) || (st = check_blob(top, "top")) ||
        (st = check_blob(top_diff, "top_diff")) || (st = check_blob(bottom_diff, "bottom_diff")))
        return st;
    const caffe_shape4& s = bottom->shape;
    if (!same_shape(s, top->shape) || !same_shape(s, top_diff->shape) || !same_shape(s, bottom_diff->shape))
        return fail(CAFFE_E_SHAPE, "LRN backward blobs must share bottom's shape");
    const caffe_dtype dt = bottom->dtype;
    if (top->dtype != dt || top_diff->dtype != dt || bottom_diff->dtype != dt) return fail(CAFFE_E_DTYPE, "LRN blobs must share one dtype");
    if (top->layout != bottom->layout || top_diff->layout != bottom->layout || bottom_diff->layout != bottom->layout)
        return fail(CAFFE_E_SHAPE, "LRN blobs must share one layout");
    if (scale) {
        if ((st = check_blob(scale, "scale"))) return st;
        if (scale->dtype != CAFFE_F32 || !same_shape(scale->shape, s) || scale->layout != bottom->layout)
            return fail(CAFFE_E_SHAPE, "scale must be F32 with bottom's shape and layout");
    }
    if (overlap(bottom_diff, bottom) || overlap(bottom_diff, top) || overlap(bottom_diff, top_diff) || overlap(bottom_diff, scale))
        return fail(CAFFE_E_ALIAS, "bottom_diff overlaps an input");
    if (s.n == 0) return CAFFE_OK;
    CK(lrn_bwd(bottom->ptr, top->ptr, top_diff->ptr, scale ? (const float*)scale->ptr : nullptr, bottom_diff->ptr,
               dt == CAFFE_BF16, nhwc(bottom), s.n, s.c, s.h, s.w, desc->local_size, desc->alpha, desc->beta, desc->k,
               (cudaStream_t)stream),
       "lrn bwd");
    return CAFFE_OK;
}

// ------------------------------------------------------------------ inner product
// bottom (N,C,H,W) is flattened to rows of K = C*H*W in the (c,h,w) order of S:130; an NHWC bottom
// with H*W > 1 and C > 1 is staged into that order.
static bool rows_direct(const caffe_blob* b, int E) {
    const bool order_ok = !nhwc(b) || (b->shape.h == 1 && b->shape.w == 1) || b->shape.c == 1;
    const long long K = (long long)b->shape.c * b->shape.h * b->shape.w;
    return order_ok && E == 2 && b->dtype == CAFFE_BF16 && aligned16(b->ptr) && (K * 2) % 16 == 0;
}
static caffe_status ip_shapes(const caffe_blob* bottom, const caffe_blob* weight, long long* K, int* O) {
    *K = (long long)bottom->shape.c * bottom->shape.h * bottom->shape.w;
    *O = weight->shape.n;
    if ((long long)weight->shape.c * weight->shape.h * weight->shape.w != *K)
        return fail(CAFFE_E_SHAPE, "weight fan-in %lld != bottom C*H*W %lld (S:183)",
                    (long long)weight->shape.c * weight->shape.h * weight->shape.w, *K);
    return CAFFE_OK;
}

// Split-K plan of an inner-product GEMM with M rows, Ncols columns and Kred reduction elements
// (kchunk per 128-byte block): the fc layers have few (M, N) tiles at batch 256, so the reduction
// is split until the units fill the SMs once; partials are reduced in a fixed order.
struct IpPlan {
    int BN, m_tiles, n_tiles, kblocks, splits, kb_per, cg;
    size_t part_bytes;
};
// cg_ok: the operand layouts allow a CTA pair (B split in halves); a pair (M = 256 rows) is used
// when the GEMM has more than 128 rows, so each weight tile is staged once for the whole batch.
static IpPlan ip_plan(long long M, long long Ncols, long long Kred, int kchunk, int BN, int E, bool cg_ok) {
    IpPlan q;
    q.BN = BN;
    q.cg = (E == 2 && cg_ok && M > 128 && g_force_cg != 1) ? 2 : 1;
    const int TM = 128 * q.cg;
    q.m_tiles = (int)cdiv(M, TM);
    q.n_tiles = (int)cdiv(Ncols, BN);
    q.kblocks = (int)cdiv(Kred, kchunk);
    q.splits = 1;
    q.kb_per = q.kblocks;
    const long long tiles = (long long)q.m_tiles * q.n_tiles;
    const int slots = 148 / q.cg;   // CTAs (or pairs) resident at once
    if (tiles < slots / 2) {
        int sp = (int)(slots / tiles);
        if (sp > q.kblocks / 4) sp = q.kblocks / 4;
        if (g_ip_max_splits > 0 && sp > g_ip_max_splits) sp = g_ip_max_splits;
        if (sp > 1) {
            q.kb_per = (int)cdiv(q.kblocks, sp);
            q.splits = (int)cdiv(q.kblocks, q.kb_per);
        }
    }
    q.part_bytes = q.splits > 1 ? align1k((size_t)q.splits * tiles * BN * TM * 4) : 0;
    return q;
}
static IpPlan ip_plan_fwd(long long N, long long K, int O, int E) {
    const int BN = (g_ip_fwd_small_bn > 0 && O <= 1024) ? g_ip_fwd_small_bn : choose_bn(O);
    return ip_plan(N, O, K, 128 / E, BN, E, (BN / 2) % 8 == 0);
}
static IpPlan ip_plan_dgrad(long long N, long long K, int O, int E) {
    const int BN = choose_bn((int)(K < 256 ? K : 256)), CH = 128 / E;
    return ip_plan(N, K, O, CH, BN, E, (BN / CH) % 2 == 0 && BN % CH == 0);
}

caffe_status caffe_ip_workspace_size(caffe_math math, caffe_shape4 bottom, int32_t O, int32_t pass, size_t* bytes) {
    if (!bytes) return fail(CAFFE_E_INVALID, "bytes is NULL");
    if (math != CAFFE_MATH_FP32 && math != CAFFE_MATH_BF16 && math != CAFFE_MATH_TF32) return fail(CAFFE_E_INVALID, "bad math mode");
    const long long N = bottom.n, K = (long long)bottom.c * bottom.h * bottom.w;
    size_t bias = align1k((size_t)bias_grad_splits((int)N, O, 1) * O * 4);
    if (math == CAFFE_MATH_FP32) { *bytes = pass == CAFFE_PASS_BACKWARD_WEIGHT ? bias : 0; return CAFFE_OK; }
    const int E = math == CAFFE_MATH_TF32 ? 4 : 2, CHh = 128 / E;
    size_t part = 0;
    if (pass == CAFFE_PASS_FORWARD && N > 0 && O > 0 && K > 0) part = ip_plan_fwd(N, K, O, E).part_bytes;
    if (pass == CAFFE_PASS_BACKWARD_DATA && N > 0 && O > 0 && K > 0) part = ip_plan_dgrad(N, K, O, E).part_bytes;
    // worst case: every operand staged (+ fp32 rows for an NHWC data gradient) + bias partials + split-K partials
    *bytes = align1k((size_t)N * rup(K, CHh) * E) + align1k((size_t)O * rup(K, CHh) * E) +
             align1k((size_t)N * rup(O, CHh) * E) + align1k((size_t)N * K * 4) + bias + part;
    return CAFFE_OK;
}

// stage a blob as (rows x cols) TMA-able rows (bf16 or tf32) into `cursor`, return pointer and ld
static cudaError_t stage_rows(const caffe_blob* b, long long rows, long long cols, int E, char*& cursor, const void** out,
                              long long* ld, cudaStream_t s) {
    if (rows_direct(b, E)) {
        *out = b->ptr;
        *ld = cols;
        return cudaSuccess;
    }
    const long long ldp = rup(cols, 128 / E);
    cudaError_t e;
    if (nhwc(b) && b->shape.h * b->shape.w > 1 && b->shape.c > 1)
        e = nhwc_to_rows(b->ptr, isbf(b), cursor, E, b->shape.n, b->shape.c, b->shape.h * b->shape.w, ldp, s);
    else
        e = convert_pad_2d(b->ptr, isbf(b), cols, cursor, E, ldp, rows, cols, s);
    *out = cursor;
    *ld = ldp;
    cursor += align1k((size_t)rows * ldp * E);
    return e;
}

caffe_status caffe_ip_forward(caffe_math math, uint32_t flags, const caffe_blob* bottom, const caffe_blob* weight,
                              const caffe_blob* bias, caffe_blob* top, void* ws, size_t ws_bytes, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom, "bottom")) || (st = check_blob(weight, "weight")) || (st = check_blob(top, "top"))) return st;
    long long K; int O;
    if ((st = ip_shapes(bottom, weight, &K, &O))) return st;
    const int N = bottom->shape.n;
    if (top->shape.n != N || top->shape.c != O || top->shape.h != 1 || top->shape.w != 1)
        return fail(CAFFE_E_SHAPE, "top must be (%d,%d,1,1)", N, O);
    if (bias) {
        if ((st = check_blob(bias, "bias"))) return st;
        if (bias->dtype != CAFFE_F32 || cnt(bias->shape) != O) return fail(CAFFE_E_SHAPE, "bias must be F32 with %d elements", O);
    }
    if (overlap(top, bottom) || overlap(top, weight) || overlap(top, bias)) return fail(CAFFE_E_ALIAS, "top overlaps an input");
    if (math == CAFFE_MATH_TF32 && (bottom->dtype == CAFFE_BF16 || weight->dtype == CAFFE_BF16 || top->dtype == CAFFE_BF16))
        return fail(CAFFE_E_DTYPE, "TF32 math with BF16 storage");
    if (math != CAFFE_MATH_FP32 && math != CAFFE_MATH_BF16 && math != CAFFE_MATH_TF32) return fail(CAFFE_E_INVALID, "bad math");
    if (N == 0) return CAFFE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int relu = (flags & CAFFE_FUSE_RELU) ? 1 : 0;
    const float* bptr = bias ? (const float*)bias->ptr : nullptr;
    if (math == CAFFE_MATH_FP32) {
        const caffe_shape4& b = bottom->shape;
        ConvGeom g{N, b.c, b.h, b.w, O, b.h, b.w, 1, 1, 0, 0, 1, 1, 1};
        L4 ly{O, 1, 1, 1};
        CK(fp32_conv_fwd(bottom->ptr, isbf(bottom), strides(bottom), weight->ptr, isbf(weight), bptr, top->ptr, isbf(top), ly,
                         1, relu, g, s),
           "ip fwd fp32");
        return CAFFE_OK;
    }
    size_t need;
    caffe_ip_workspace_size(math, bottom->shape, O, 0, &need);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    const int E = math == CAFFE_MATH_TF32 ? 4 : 2;
    char* cur = (char*)ws;
    const void *A, *B;
    long long lda, ldb;
    CK(stage_rows(bottom, N, K, E, cur, &A, &lda, s), "stage bottom");
    CK(stage_rows(weight, O, K, E, cur, &B, &ldb, s), "stage weight");
    TcLaunch L;
    memset(&L, 0, sizeof L);
    const IpPlan q = ip_plan_fwd(N, K, O, E);
    float* part = nullptr;
    if (q.splits > 1) { part = (float*)cur; cur += q.part_bytes; }
    L.esz = E; L.amode = A_TILED_K; L.bmode = B_TILED_K; L.epi = q.splits > 1 ? EPI_PARTIAL : EPI_STRIDED;
    L.cg = q.cg;
    TcArgs& a = L.args;
    a.BN = q.BN;
    if (!encode_tiled_2d(&L.mapA, E, A, lda, N, lda * E, 128 / E, 128) ||
        !encode_tiled_2d(&L.mapB, E, B, ldb, O, ldb * E, 128 / E, a.BN / q.cg))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (ip fwd)");
    a.M = N; a.N = O; a.m_tiles = q.m_tiles; a.n_tiles = q.n_tiles; a.groups = 1; a.splits = q.splits;
    a.kblocks = q.kblocks; a.kb_per_split = q.kb_per;
    a.out = top->ptr; a.out_bf16 = isbf(top); a.s_n = O; a.s_c = 1; a.s_p = 0; a.P = 1; a.col_g = 0;
    a.bias = bptr; a.relu = relu; a.beta = 0.f; a.partial = part;
    finish_args(a, a.BN / q.cg * 128);
    if (!part) enable_tma_store(L, top->ptr, isbf(top) ? 2 : 4, O, N, O, true);
    if ((st = run_tc(L, s, 2.0 * N * O * (double)K, 1))) return st;
    if (part)
        CK(gemm_partial_reduce(part, q.splits, q.m_tiles, q.n_tiles, q.BN, 128 * q.cg, N, O, top->ptr, isbf(top), O, bptr,
                               relu, 0.f, 0, 0, s),
           "ip fwd split-K reduce");
    return CAFFE_OK;
}

static caffe_status ip_bwd_data(caffe_math math, const caffe_blob* top_diff, const caffe_blob* weight,
                                const caffe_blob* relu_top, caffe_blob* bottom_diff, float beta, void* ws, size_t ws_bytes,
                                caffe_stream_t stream);

caffe_status caffe_ip_backward_data(caffe_math math, const caffe_blob* top_diff, const caffe_blob* weight,
                                    caffe_blob* bottom_diff, float beta, void* ws, size_t ws_bytes, caffe_stream_t stream) {
    return ip_bwd_data(math, top_diff, weight, nullptr, bottom_diff, beta, ws, ws_bytes, stream);
}

caffe_status caffe_ip_backward_data_relu(caffe_math math, const caffe_blob* top_diff, const caffe_blob* weight,
                                         const caffe_blob* relu_top, caffe_blob* bottom_diff, void* ws, size_t ws_bytes,
                                         caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(relu_top, "relu_top"))) return st;
    if ((st = check_blob(bottom_diff, "bottom_diff"))) return st;
    if (!same_shape(relu_top->shape, bottom_diff->shape))
        return fail(CAFFE_E_SHAPE, "relu_top shape (%d,%d,%d,%d) != bottom_diff shape (%d,%d,%d,%d)", relu_top->shape.n,
                    relu_top->shape.c, relu_top->shape.h, relu_top->shape.w, bottom_diff->shape.n, bottom_diff->shape.c,
                    bottom_diff->shape.h, bottom_diff->shape.w);
    if (nhwc(relu_top) != nhwc(bottom_diff)) return fail(CAFFE_E_INVALID, "relu_top and bottom_diff layouts differ");
    if (overlap(bottom_diff, relu_top)) return fail(CAFFE_E_ALIAS, "bottom_diff overlaps relu_top");
    return ip_bwd_data(math, top_diff, weight, relu_top, bottom_diff, 0.f, ws, ws_bytes, stream);
}

static caffe_status ip_bwd_data(caffe_math math, const caffe_blob* top_diff, const caffe_blob* weight,
                                const caffe_blob* relu_top, caffe_blob* bottom_diff, float beta, void* ws, size_t ws_bytes,
                                caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(top_diff, "top_diff")) || (st = check_blob(weight, "weight")) ||
        (st = check_blob(bottom_diff, "bottom_diff")))
        return st;
    long long K; int O;
    if ((st = ip_shapes(bottom_diff, weight, &K, &O))) return st;
    const int N = bottom_diff->shape.n;
    if (top_diff->shape.n != N || top_diff->shape.c != O || top_diff->shape.h != 1 || top_diff->shape.w != 1)
        return fail(CAFFE_E_SHAPE, "top_diff must be (%d,%d,1,1)", N, O);
    if (overlap(bottom_diff, top_diff) || overlap(bottom_diff, weight)) return fail(CAFFE_E_ALIAS, "bottom_diff overlaps an input");
    if (math == CAFFE_MATH_TF32 && (top_diff->dtype == CAFFE_BF16 || weight->dtype == CAFFE_BF16))
        return fail(CAFFE_E_DTYPE, "TF32 math with BF16 storage");
    if (math != CAFFE_MATH_FP32 && math != CAFFE_MATH_BF16 && math != CAFFE_MATH_TF32) return fail(CAFFE_E_INVALID, "bad math");
    if (N == 0) return CAFFE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const caffe_shape4& xs = bottom_diff->shape;
    if (math == CAFFE_MATH_FP32) {   // CUDA-core FP32 FMA
        ConvGeom g{N, xs.c, xs.h, xs.w, O, xs.h, xs.w, 1, 1, 0, 0, 1, 1, 1};
        L4 ly{O, 1, 1, 1};
        CK(fp32_conv_dgrad(top_diff->ptr, isbf(top_diff), ly, weight->ptr, isbf(weight), bottom_diff->ptr,
                           isbf(bottom_diff), nhwc(bottom_diff), beta, g, s, 0),
           "ip dgrad fp32");
        if (relu_top)
            CK(relu_bwd(relu_top->ptr, bottom_diff->ptr, bottom_diff->ptr, isbf(relu_top), isbf(bottom_diff),
                        (int)((long long)N * K), s),
               "relu backward");
        return CAFFE_OK;
    }
    size_t need;
    caffe_ip_workspace_size(math, bottom_diff->shape, O, 1, &need);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    // BF16, or TF32 (tcgen05 kind::tf32; operands staged TF32-RN, the MN-major weight tile too)
    const int E = math == CAFFE_MATH_TF32 ? 4 : 2, CH = 128 / E;
    char* cur = (char*)ws;
    const void *A, *B;
    long long lda, ldb;
    CK(stage_rows(top_diff, N, O, E, cur, &A, &lda, s), "stage top_diff");
    CK(stage_rows(weight, O, K, E, cur, &B, &ldb, s), "stage weight");
    const bool permute = nhwc(bottom_diff) && xs.h * xs.w > 1 && xs.c > 1;
    const IpPlan q = ip_plan_dgrad(N, K, O, E);
    float* part = nullptr;
    if (q.splits > 1) { part = (float*)cur; cur += q.part_bytes; }
    float* rows = permute && !part ? (float*)cur : nullptr;
    TcLaunch L;
    memset(&L, 0, sizeof L);
    L.esz = E; L.amode = A_TILED_K; L.bmode = B_TILED_MN; L.epi = part ? EPI_PARTIAL : EPI_STRIDED;
    L.cg = q.cg;
    TcArgs& a = L.args;
    a.BN = q.BN;
    if (!encode_tiled_2d(&L.mapA, E, A, lda, N, lda * E, CH, 128) ||
        !encode_tiled_2d(&L.mapB, E, B, ldb, O, ldb * E, CH, CH, E == 4))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (ip dgrad)");
    a.M = N; a.N = (int)K; a.m_tiles = q.m_tiles; a.n_tiles = q.n_tiles; a.groups = 1; a.splits = q.splits;
    a.kblocks = q.kblocks; a.kb_per_split = q.kb_per; a.b_nchunks = (int)cdiv(a.BN, CH);
    a.partial = part;
    if (rows) {
        a.out = rows; a.out_bf16 = 0; a.beta = 0.f;
    } else {
        a.out = bottom_diff->ptr; a.out_bf16 = isbf(bottom_diff); a.beta = beta;
    }
    a.s_n = K; a.s_c = 1; a.s_p = 0; a.P = 1;
    // ReLU backward folded in (beta is 0 then): in the split-K reduce (row-major output), in the
    // tensor-core epilogue (direct output), else by a separate in-place pass
    bool masked = false;
    if (relu_top && !part && !rows) {
        a.relu_top = relu_top->ptr; a.relu_top_bf16 = isbf(relu_top);
        masked = true;
    }
    finish_args(a, a.b_nchunks / q.cg * CH * 128);
    if (!part && (!masked || (a.out_bf16 && a.relu_top_bf16 && K % 64 == 0)))
        enable_tma_store(L, a.out, a.out_bf16 ? 2 : 4, K, N, K, true);
    if ((st = run_tc(L, s, 2.0 * N * O * (double)K, 1))) return st;
    if (part) {
        const bool mred = relu_top && !permute;
        cudaError_t e = gemm_partial_reduce(part, q.splits, q.m_tiles, q.n_tiles, q.BN, 128 * q.cg, N, (int)K,
                                            bottom_diff->ptr, isbf(bottom_diff), K, nullptr, 0, beta, permute ? xs.c : 0,
                                            xs.h * xs.w, s, mred ? relu_top->ptr : nullptr, mred ? isbf(relu_top) : 0);
        if (e == cudaErrorNotSupported && mred) {   // no masked form for this layout: plain reduce + ReLU pass
            e = gemm_partial_reduce(part, q.splits, q.m_tiles, q.n_tiles, q.BN, 128 * q.cg, N, (int)K, bottom_diff->ptr,
                                    isbf(bottom_diff), K, nullptr, 0, beta, 0, xs.h * xs.w, s);
            if (e == cudaSuccess) masked = false;
        } else if (mred) {
            masked = true;
        }
        CK(e, "ip dgrad split-K reduce");
    } else if (rows) {
        CK(rows_to_nhwc(rows, K, bottom_diff->ptr, isbf(bottom_diff), N, xs.c, xs.h * xs.w, beta, s), "ip dgrad to NHWC");
    }
    if (relu_top && !masked)
        CK(relu_bwd(relu_top->ptr, bottom_diff->ptr, bottom_diff->ptr, isbf(relu_top), isbf(bottom_diff),
                    (int)((long long)N * K), s),
           "relu backward");
    return CAFFE_OK;
}

caffe_status caffe_ip_backward_weight(caffe_math math, const caffe_blob* bottom, const caffe_blob* top_diff,
                                      caffe_blob* weight_diff, caffe_blob* bias_diff, float beta, void* ws, size_t ws_bytes,
                                      caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom, "bottom")) || (st = check_blob(top_diff, "top_diff")) ||
        (st = check_blob(weight_diff, "weight_diff")))
        return st;
    long long K; int O;
    if ((st = ip_shapes(bottom, weight_diff, &K, &O))) return st;
    const int N = bottom->shape.n;
    if (top_diff->shape.n != N || top_diff->shape.c != O || top_diff->shape.h != 1 || top_diff->shape.w != 1)
        return fail(CAFFE_E_SHAPE, "top_diff must be (%d,%d,1,1)", N, O);
    if (weight_diff->dtype != CAFFE_F32) return fail(CAFFE_E_DTYPE, "weight_diff must be F32");
    if (bias_diff) {
        if ((st = check_blob(bias_diff, "bias_diff"))) return st;
        if (bias_diff->dtype != CAFFE_F32 || cnt(bias_diff->shape) != O) return fail(CAFFE_E_SHAPE, "bias_diff must be F32 with %d elements", O);
    }
    if (overlap(weight_diff, bottom) || overlap(weight_diff, top_diff) || overlap(bias_diff, bottom) ||
        overlap(bias_diff, top_diff) || overlap(bias_diff, weight_diff))
        return fail(CAFFE_E_ALIAS, "weight_diff/bias_diff overlaps an input");
    if (math == CAFFE_MATH_TF32 && (top_diff->dtype == CAFFE_BF16 || bottom->dtype == CAFFE_BF16))
        return fail(CAFFE_E_DTYPE, "TF32 math with BF16 storage");
    if (math != CAFFE_MATH_FP32 && math != CAFFE_MATH_BF16 && math != CAFFE_MATH_TF32) return fail(CAFFE_E_INVALID, "bad math");
    if (N == 0) return CAFFE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    size_t need;
    caffe_ip_workspace_size(math, bottom->shape, O, CAFFE_PASS_BACKWARD_WEIGHT, &need);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    char* cur = (char*)ws;
    float* bpart = (float*)cur;
    cur += align1k((size_t)bias_grad_splits(N, O, 1) * O * 4);
    if (bias_diff) CK(bias_grad(top_diff->ptr, isbf(top_diff), 1, (float*)bias_diff->ptr, beta, N, O, 1, bpart, s), "ip bias grad");
    if (math == CAFFE_MATH_FP32) {   // CUDA-core FP32 FMA (blocked reduction, R13)
        const caffe_shape4& b = bottom->shape;
        ConvGeom g{N, b.c, b.h, b.w, O, b.h, b.w, 1, 1, 0, 0, 1, 1, 1};
        L4 ly{O, 1, 1, 1};
        CK(fp32_conv_wgrad(bottom->ptr, isbf(bottom), strides(bottom), top_diff->ptr, isbf(top_diff), ly,
                           (float*)weight_diff->ptr, beta, g, s, 0),
           "ip wgrad fp32");
        return CAFFE_OK;
    }
    // BF16, or TF32 (tcgen05 kind::tf32 with both operands MN-major, staged TF32-RN)
    const int E = math == CAFFE_MATH_TF32 ? 4 : 2, CH = 128 / E;
    const void *A, *B;
    long long lda, ldb;
    CK(stage_rows(top_diff, N, O, E, cur, &A, &lda, s), "stage top_diff");
    CK(stage_rows(bottom, N, K, E, cur, &B, &ldb, s), "stage bottom");
    TcLaunch L;
    memset(&L, 0, sizeof L);
    // dW tiles: M runs over the outputs o, N over the fan-in k; each epilogue thread writes 16
    // consecutive k of its dW row as float4 vectors (measured faster than the transposed,
    // lane-coalesced layout); the reduction runs over the batch.
    L.esz = E; L.amode = A_TILED_MN; L.bmode = B_TILED_MN; L.epi = EPI_STRIDED;
    TcArgs& a = L.args;
    a.BN = choose_bn((int)(K < 256 ? K : 256));
    // CTA pairs (M = 256 output rows) stage each bottom tile once for 256 outputs
    L.cg = (E == 2 && O > 128 && a.BN % 128 == 0 && g_force_cg != 1) ? 2 : 1;
    if (!encode_tiled_2d(&L.mapA, E, A, lda, N, lda * E, CH, CH, E == 4) ||
        !encode_tiled_2d(&L.mapB, E, B, ldb, N, ldb * E, CH, CH, E == 4))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (ip wgrad)");
    a.M = O; a.N = (int)K; a.m_tiles = (int)cdiv(O, 128 * L.cg); a.n_tiles = (int)cdiv(K, a.BN); a.groups = 1;
    a.splits = 1;
    a.kblocks = (int)cdiv(N, CH); a.kb_per_split = a.kblocks; a.b_nchunks = (int)cdiv(a.BN, CH);
    a.out = weight_diff->ptr; a.out_bf16 = 0; a.s_n = K; a.s_c = 1; a.s_p = 0; a.P = 1; a.beta = beta;
    finish_args(a, a.b_nchunks / L.cg * CH * 128);
    enable_tma_store(L, weight_diff->ptr, 4, K, O, K, true);
    return run_tc(L, s, 2.0 * N * O * (double)K, 1);
}

caffe_status caffe_ip_backward_weight_sgd(const caffe_blob* bottom, const caffe_blob* top_diff, caffe_blob* weight,
                                          caffe_blob* momentum, caffe_blob* weight_bf16, caffe_blob* bias_diff, float lr,
                                          float mom, float decay, float grad_scale, void* ws, size_t ws_bytes,
                                          caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom, "bottom")) || (st = check_blob(top_diff, "top_diff")) ||
        (st = check_blob(weight, "weight")) || (st = check_blob(momentum, "momentum")) ||
        (st = check_blob(weight_bf16, "weight_bf16")))
        return st;
    long long K; int O;
    if ((st = ip_shapes(bottom, weight, &K, &O))) return st;
    const int N = bottom->shape.n;
    if (top_diff->shape.n != N || top_diff->shape.c != O || top_diff->shape.h != 1 || top_diff->shape.w != 1)
        return fail(CAFFE_E_SHAPE, "top_diff must be (%d,%d,1,1)", N, O);
    if (weight->dtype != CAFFE_F32 || momentum->dtype != CAFFE_F32 || weight_bf16->dtype != CAFFE_BF16)
        return fail(CAFFE_E_DTYPE, "weight and momentum must be F32, weight_bf16 BF16");
    if (!same_shape(momentum->shape, weight->shape) || !same_shape(weight_bf16->shape, weight->shape))
        return fail(CAFFE_E_SHAPE, "momentum and weight_bf16 must have the weight's shape");
    if (nhwc(weight) || nhwc(momentum) || nhwc(weight_bf16)) return fail(CAFFE_E_INVALID, "weights must be row-major (O, K)");
    if (K % 32 != 0 || !aligned16(weight->ptr) || !aligned16(momentum->ptr) || !aligned16(weight_bf16->ptr))
        return fail(CAFFE_E_ALIGN, "fused update needs K %% 32 == 0 and 16-byte aligned weights (K = %lld)", K);
    if (bias_diff) {
        if ((st = check_blob(bias_diff, "bias_diff"))) return st;
        if (bias_diff->dtype != CAFFE_F32 || cnt(bias_diff->shape) != O) return fail(CAFFE_E_SHAPE, "bias_diff must be F32 with %d elements", O);
    }
    if (overlap(weight, bottom) || overlap(weight, top_diff) || overlap(momentum, weight) || overlap(weight_bf16, weight) ||
        overlap(weight_bf16, momentum) || overlap(weight_bf16, bottom) || overlap(weight_bf16, top_diff))
        return fail(CAFFE_E_ALIAS, "weight / momentum / weight_bf16 overlap each other or an input");
    if (N == 0) return CAFFE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    size_t need;
    caffe_ip_workspace_size(CAFFE_MATH_BF16, bottom->shape, O, CAFFE_PASS_BACKWARD_WEIGHT, &need);
    if ((st = check_ws(ws, ws_bytes, need))) return st;
    char* cur = (char*)ws;
    float* bpart = (float*)cur;
    cur += align1k((size_t)bias_grad_splits(N, O, 1) * O * 4);
    if (bias_diff) CK(bias_grad(top_diff->ptr, isbf(top_diff), 1, (float*)bias_diff->ptr, 0.f, N, O, 1, bpart, s), "ip bias grad");
    const int E = 2;
    const void *A, *B;
    long long lda, ldb;
    CK(stage_rows(top_diff, N, O, E, cur, &A, &lda, s), "stage top_diff");
    CK(stage_rows(bottom, N, K, E, cur, &B, &ldb, s), "stage bottom");
    TcLaunch L;
    memset(&L, 0, sizeof L);
    L.esz = E; L.amode = A_TILED_MN; L.bmode = B_TILED_MN; L.epi = EPI_STRIDED;
    TcArgs& a = L.args;
    a.BN = choose_bn((int)(K < 256 ? K : 256));
    L.cg = (O > 128 && a.BN % 128 == 0 && g_force_cg != 1) ? 2 : 1;
    if (!encode_tiled_2d(&L.mapA, E, A, lda, N, lda * E, 64, 64) || !encode_tiled_2d(&L.mapB, E, B, ldb, N, ldb * E, 64, 64))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (ip wgrad sgd)");
    a.M = O; a.N = (int)K; a.m_tiles = (int)cdiv(O, 128 * L.cg); a.n_tiles = (int)cdiv(K, a.BN); a.groups = 1;
    a.splits = 1;
    a.kblocks = (int)cdiv(N, 64); a.kb_per_split = a.kblocks; a.b_nchunks = (int)cdiv(a.BN, 64);
    a.out = weight->ptr; a.out_bf16 = 0; a.s_n = K; a.s_c = 1; a.s_p = 0; a.P = 1; a.beta = 0.f;
    L.epi = EPI_SGD;
    a.sgd = 1; a.sgd_v = (float*)momentum->ptr;
    a.sgd_lr = lr; a.sgd_mom = mom; a.sgd_decay = decay; a.sgd_gs = grad_scale;
    finish_args(a, a.b_nchunks / L.cg * 64 * 128);
    if (!encode_store_2d(&L.mapC, 4, weight->ptr, K, O, K) || !encode_store_2d(&L.mapV, 4, momentum->ptr, K, O, K) ||
        !encode_store_2d_bf16_32(&L.mapWb, weight_bf16->ptr, K, O, K))
        return fail(CAFFE_E_CUDA, "cuTensorMapEncodeTiled failed (fused update stores)");
    a.tma_store = 1;
    // stages: the SGD staging (80 KB) leaves ~130 KB for the operand ring
    const int stage = (a.macc > 1 ? a.macc : 1) * 16384 + a.b_stage_bytes;
    a.stages = std::max(2, std::min(a.stages, (227 * 1024 - 80 * 1024 - 8 * 1024) / stage));
    return run_tc(L, s, 2.0 * N * O * (double)K, 1);
}

caffe_status caffe_blob_to_nchw(const caffe_blob* src, caffe_blob* dst, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(src, "src")) || (st = check_blob(dst, "dst"))) return st;
    if (!same_shape(src->shape, dst->shape)) return fail(CAFFE_E_SHAPE, "src and dst shapes differ");
    if (!nhwc(src) || nhwc(dst)) return fail(CAFFE_E_INVALID, "src must be channels-last and dst NCHW");
    if (overlap(src, dst)) return fail(CAFFE_E_ALIAS, "dst overlaps src");
    if (dst->dtype != CAFFE_BF16) return fail(CAFFE_E_DTYPE, "dst must be BF16 (F32 rows are staged TF32-rounded)");
    const caffe_shape4& b = src->shape;
    if (b.n == 0) return CAFFE_OK;
    CK(nhwc_to_rows(src->ptr, isbf(src), dst->ptr, isbf(dst) ? 2 : 4, b.n, b.c, b.h * b.w, (long long)b.c * b.h * b.w,
                    (cudaStream_t)stream),
       "nhwc to nchw");
    return CAFFE_OK;
}

// ------------------------------------------------------------------ im2col / col2im
caffe_status caffe_im2col(const caffe_conv_desc* desc, const caffe_blob* bottom, int32_t n, caffe_blob* col,
                          caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom, "bottom")) || (st = check_blob(col, "col"))) return st;
    if (bottom->dtype != CAFFE_F32 || col->dtype != CAFFE_F32) return fail(CAFFE_E_DTYPE, "im2col is F32 only");
    if (nhwc(bottom) || nhwc(col)) return fail(CAFFE_E_INVALID, "im2col is defined on NCHW blobs (S:297)");
    if (!desc) return fail(CAFFE_E_INVALID, "desc is NULL");
    caffe_conv_desc d = *desc;
    d.group = 1;
    Plan p;
    if ((st = conv_validate(&d, bottom->shape, 1, &p))) return st;
    if (n < 0 || n >= bottom->shape.n) return fail(CAFFE_E_PARAM, "image index %d out of range", n);
    if (cnt(col->shape) != (long long)p.C * p.kh * p.kw * p.OH * p.OW) return fail(CAFFE_E_SHAPE, "col must hold C*kh*kw*OH*OW elements");
    if (overlap(col, bottom)) return fail(CAFFE_E_ALIAS, "col overlaps bottom");
    CK(im2col_k((const float*)bottom->ptr, n, cgeom(p), (float*)col->ptr, (cudaStream_t)stream), "im2col");
    return CAFFE_OK;
}

caffe_status caffe_col2im(const caffe_conv_desc* desc, const caffe_blob* col, int32_t n, caffe_blob* bottom_diff,
                          caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom_diff, "bottom_diff")) || (st = check_blob(col, "col"))) return st;
    if (bottom_diff->dtype != CAFFE_F32 || col->dtype != CAFFE_F32) return fail(CAFFE_E_DTYPE, "col2im is F32 only");
    if (nhwc(bottom_diff) || nhwc(col)) return fail(CAFFE_E_INVALID, "col2im is defined on NCHW blobs (S:297)");
    if (!desc) return fail(CAFFE_E_INVALID, "desc is NULL");
    caffe_conv_desc d = *desc;
    d.group = 1;
    Plan p;
    if ((st = conv_validate(&d, bottom_diff->shape, 1, &p))) return st;
    if (n < 0 || n >= bottom_diff->shape.n) return fail(CAFFE_E_PARAM, "image index %d out of range", n);
    if (cnt(col->shape) != (long long)p.C * p.kh * p.kw * p.OH * p.OW) return fail(CAFFE_E_SHAPE, "col must hold C*kh*kw*OH*OW elements");
    if (overlap(col, bottom_diff)) return fail(CAFFE_E_ALIAS, "col overlaps bottom_diff");
    CK(col2im_k((const float*)col->ptr, n, cgeom(p), (float*)bottom_diff->ptr, (cudaStream_t)stream), "col2im");
    return CAFFE_OK;
}

// ------------------------------------------------------------------ glue
caffe_status caffe_softmax_loss(const caffe_blob* scores, const int32_t* labels, float* loss, caffe_blob* score_diff,
                                caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(scores, "scores"))) return st;
    if (!labels || !loss) return fail(CAFFE_E_INVALID, "labels and loss are required");
    const int N = scores->shape.n;
    const long long K = (long long)scores->shape.c * scores->shape.h * scores->shape.w;
    if (scores->shape.h * scores->shape.w != 1 && nhwc(scores)) return fail(CAFFE_E_INVALID, "scores must be (N,K,1,1) or NCHW");
    if (score_diff) {
        if ((st = check_blob(score_diff, "score_diff"))) return st;
        if (!same_shape(score_diff->shape, scores->shape)) return fail(CAFFE_E_SHAPE, "score_diff must match scores");
        if (score_diff->shape.h * score_diff->shape.w != 1 && nhwc(score_diff)) return fail(CAFFE_E_INVALID, "score_diff must be NCHW");
        if (overlap(score_diff, scores)) return fail(CAFFE_E_ALIAS, "score_diff overlaps scores");
    }
    if (N == 0) return CAFFE_OK;
    CK(softmax_loss_k(scores->ptr, isbf(scores), labels, loss, score_diff ? score_diff->ptr : nullptr,
                      score_diff ? isbf(score_diff) : 0, N, (int)K, (cudaStream_t)stream),
       "softmax loss");
    return CAFFE_OK;
}

caffe_status caffe_sgd_update(float* w, const float* g, float* v, void* w_bf16, int64_t count, float lr, float momentum,
                              float decay, float grad_scale, caffe_stream_t stream) {
    if (count < 0) return fail(CAFFE_E_SHAPE, "negative count");
    if (count == 0) return CAFFE_OK;
    if (!w || !g || !v) return fail(CAFFE_E_INVALID, "w, g and v are required");
    if (!aligned16(w) || !aligned16(g) || !aligned16(v) || (reinterpret_cast<uintptr_t>(w_bf16) & 7))
        return fail(CAFFE_E_ALIGN, "SGD buffers must be 16-byte aligned (w_bf16 8-byte)");
    CK(sgd_k(w, g, v, w_bf16, count, lr, momentum, decay, grad_scale, (cudaStream_t)stream), "sgd update");
    return CAFFE_OK;
}


// ------------------------------------------------------------------ fused pool + LRN (NEXT-1)
static caffe_status pool_lrn_check(const caffe_pool_desc* pd, const caffe_lrn_desc* ld, const caffe_blob* bottom_like,
                                   const caffe_blob* pooled, const caffe_blob* mask, PoolGeom* g) {
    caffe_status st;
    if ((st = lrn_validate(ld))) return st;
    if ((st = check_blob(bottom_like, "bottom")) || (st = check_blob(pooled, "pool_top"))) return st;
    if ((st = check_blob(mask, "mask", false))) return st;
    if ((st = pool_validate(pd, bottom_like->shape, g))) return st;
    if (pd->method != CAFFE_POOL_MAX) return fail(CAFFE_E_INVALID, "the fused kernels pool with MAX");
    caffe_shape4 want{g->N, g->C, g->OH, g->OW};
    if (!same_shape(pooled->shape, want) || !same_shape(mask->shape, want))
        return fail(CAFFE_E_SHAPE, "pool_top and mask must be (%d,%d,%d,%d)", want.n, want.c, want.h, want.w);
    if (!isbf(bottom_like) || !isbf(pooled) || !nhwc(bottom_like) || !nhwc(pooled) || !nhwc(mask) ||
        mask->dtype != CAFFE_U8)
        return fail(CAFFE_E_DTYPE, "the fused pool+LRN kernels take BF16 channels-last blobs and a U8 mask");
    if (!pool_lrn_fusable(*g, ld->local_size))
        return fail(CAFFE_E_INVALID, "the fused pool+LRN kernels need 3x3/s2 unpadded windows inside the map, "
                                     "C %% 8 == 0 and local_size <= 9 (use the separate calls)");
    if (!aligned16(bottom_like->ptr) || !aligned16(pooled->ptr) || !aligned16(mask->ptr))
        return fail(CAFFE_E_ALIGN, "fused pool+LRN buffers must be 16-byte aligned");
    return CAFFE_OK;
}

caffe_status caffe_pool_lrn_forward(const caffe_pool_desc* pool, const caffe_lrn_desc* lrn, const caffe_blob* bottom,
                                    caffe_blob* pool_top, caffe_blob* mask, caffe_blob* top, caffe_stream_t stream) {
    caffe_status st;
    PoolGeom g;
    if ((st = pool_lrn_check(pool, lrn, bottom, pool_top, mask, &g))) return st;
    if ((st = check_blob(top, "top"))) return st;
    if (!same_shape(top->shape, pool_top->shape) || top->dtype != pool_top->dtype || top->layout != pool_top->layout)
        return fail(CAFFE_E_SHAPE, "top must match pool_top (shape, dtype, layout)");
    if (!aligned16(top->ptr)) return fail(CAFFE_E_ALIGN, "top must be 16-byte aligned");
    if (overlap(pool_top, bottom) || overlap(mask, bottom) || overlap(top, bottom) || overlap(top, pool_top) ||
        overlap(mask, pool_top) || overlap(mask, top))
        return fail(CAFFE_E_ALIAS, "fused pool+LRN outputs overlap each other or the input");
    if (g.N == 0) return CAFFE_OK;
    CK(pool_lrn_fwd(bottom->ptr, pool_top->ptr, mask->ptr, top->ptr, g, lrn->local_size, lrn->alpha, lrn->beta, lrn->k,
                    (cudaStream_t)stream),
       "fused pool+lrn fwd");
    return CAFFE_OK;
}

caffe_status caffe_lrn_pool_backward(const caffe_pool_desc* pool, const caffe_lrn_desc* lrn, const caffe_blob* pool_top,
                                     const caffe_blob* top_diff, const caffe_blob* mask, int32_t relu,
                                     caffe_blob* bottom_diff, caffe_stream_t stream) {
    caffe_status st;
    PoolGeom g;
    if ((st = pool_lrn_check(pool, lrn, bottom_diff, pool_top, mask, &g))) return st;
    if ((st = check_blob(top_diff, "top_diff"))) return st;
    if (!same_shape(top_diff->shape, pool_top->shape) || top_diff->dtype != pool_top->dtype ||
        top_diff->layout != pool_top->layout)
        return fail(CAFFE_E_SHAPE, "top_diff must match pool_top (shape, dtype, layout)");
    if (!aligned16(top_diff->ptr)) return fail(CAFFE_E_ALIGN, "top_diff must be 16-byte aligned");
    if (overlap(bottom_diff, pool_top) || overlap(bottom_diff, top_diff) || overlap(bottom_diff, mask))
        return fail(CAFFE_E_ALIAS, "bottom_diff overlaps an input");
    if (g.N == 0) return CAFFE_OK;
    CK(lrn_pool_bwd(pool_top->ptr, top_diff->ptr, mask->ptr, bottom_diff->ptr, relu ? 1 : 0, g, lrn->local_size,
                    lrn->alpha, lrn->beta, lrn->k, (cudaStream_t)stream),
       "fused lrn+pool bwd");
    return CAFFE_OK;
}

// ------------------------------------------------------------------ catalogue layers (catalog.cu)
static caffe_status same_elementwise(const caffe_blob* a, const caffe_blob* b, const char* what) {
    if (!same_shape(a->shape, b->shape) || a->dtype != b->dtype || a->layout != b->layout)
        return fail(CAFFE_E_SHAPE, "%s must match in shape, dtype and layout", what);
    return CAFFE_OK;
}

caffe_status caffe_sigmoid_forward(const caffe_blob* bottom, caffe_blob* top, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(bottom, "bottom")) || (st = check_blob(top, "top"))) return st;
    if ((st = same_elementwise(bottom, top, "top and bottom"))) return st;
    if (bottom->ptr != top->ptr && overlap(bottom, top)) return fail(CAFFE_E_ALIAS, "partial overlap of top and bottom");
    if (cnt(bottom->shape) == 0) return CAFFE_OK;
    if (!aligned16(bottom->ptr) || !aligned16(top->ptr)) return fail(CAFFE_E_ALIGN, "sigmoid buffers must be 16-byte aligned");
    CK(sigmoid_fwd_k(bottom->ptr, top->ptr, isbf(bottom), cnt(bottom->shape), (cudaStream_t)stream), "sigmoid fwd");
    return CAFFE_OK;
}

caffe_status caffe_sigmoid_backward(const caffe_blob* top, const caffe_blob* top_diff, caffe_blob* bottom_diff,
                                    caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(top, "top")) || (st = check_blob(top_diff, "top_diff")) ||
        (st = check_blob(bottom_diff, "bottom_diff")))
        return st;
    if ((st = same_elementwise(top_diff, bottom_diff, "top_diff and bottom_diff"))) return st;
    if (!same_shape(top->shape, top_diff->shape) || top->layout != top_diff->layout)
        return fail(CAFFE_E_SHAPE, "top must match top_diff in shape and layout");
    if ((bottom_diff->ptr != top_diff->ptr && overlap(bottom_diff, top_diff)) || overlap(bottom_diff, top))
        return fail(CAFFE_E_ALIAS, "bottom_diff overlaps an input");
    if (cnt(top->shape) == 0) return CAFFE_OK;
    if (!aligned16(top->ptr) || !aligned16(top_diff->ptr) || !aligned16(bottom_diff->ptr))
        return fail(CAFFE_E_ALIGN, "sigmoid buffers must be 16-byte aligned");
    CK(sigmoid_bwd_k(top->ptr, top_diff->ptr, bottom_diff->ptr, isbf(top), isbf(top_diff), cnt(top->shape),
                     (cudaStream_t)stream),
       "sigmoid bwd");
    return CAFFE_OK;
}

static caffe_status eltwise_check(int32_t op, int32_t n, const caffe_blob* const* in, const caffe_blob* ref,
                                  bool need_inputs) {
    caffe_status st;
    if (op != CAFFE_ELTWISE_PROD && op != CAFFE_ELTWISE_SUM && op != CAFFE_ELTWISE_MAX)
        return fail(CAFFE_E_INVALID, "bad eltwise op %d", op);
    if (n < 2 || n > CAFFE_ELTWISE_MAX_INPUTS)
        return fail(CAFFE_E_PARAM, "eltwise takes 2..%d inputs (S:236), got %d", CAFFE_ELTWISE_MAX_INPUTS, n);
    if (!need_inputs) return CAFFE_OK;
    if (!in) return fail(CAFFE_E_INVALID, "inputs is NULL");
    for (int i = 0; i < n; i++) {
        if ((st = check_blob(in[i], "input"))) return st;
        if (!same_shape(in[i]->shape, ref->shape))
            return fail(CAFFE_E_SHAPE, "eltwise input %d shape (%d,%d,%d,%d) differs from (%d,%d,%d,%d)", i,
                        in[i]->shape.n, in[i]->shape.c, in[i]->shape.h, in[i]->shape.w, ref->shape.n, ref->shape.c,
                        ref->shape.h, ref->shape.w);
        if ((st = same_elementwise(in[i], ref, "eltwise inputs and outputs"))) return st;
        if (!aligned16(in[i]->ptr)) return fail(CAFFE_E_ALIGN, "eltwise input %d must be 16-byte aligned", i);
    }
    return CAFFE_OK;
}

caffe_status caffe_eltwise_forward(int32_t op, int32_t n_inputs, const caffe_blob* const* inputs, const float* coeffs,
                                   caffe_blob* top, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(top, "top"))) return st;
    if ((st = eltwise_check(op, n_inputs, inputs, top, true))) return st;
    if (coeffs && op != CAFFE_ELTWISE_SUM) return fail(CAFFE_E_PARAM, "coefficients apply to SUM only");
    for (int i = 0; i < n_inputs; i++)
        if (overlap(inputs[i], top) && inputs[i]->ptr != top->ptr)
            return fail(CAFFE_E_ALIAS, "top partially overlaps input %d", i);
    if (cnt(top->shape) == 0) return CAFFE_OK;
    if (!aligned16(top->ptr)) return fail(CAFFE_E_ALIGN, "top must be 16-byte aligned");
    const void* ptrs[CAFFE_ELTWISE_MAX_INPUTS];
    for (int i = 0; i < n_inputs; i++) ptrs[i] = inputs[i]->ptr;
    CK(eltwise_fwd_k(op, n_inputs, ptrs, coeffs, top->ptr, isbf(top), cnt(top->shape), (cudaStream_t)stream),
       "eltwise fwd");
    return CAFFE_OK;
}

caffe_status caffe_eltwise_backward(int32_t op, int32_t n_inputs, const caffe_blob* const* inputs, const float* coeffs,
                                    const caffe_blob* top_diff, caffe_blob* const* bottom_diffs, caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(top_diff, "top_diff"))) return st;
    const bool need_x = op != CAFFE_ELTWISE_SUM;
    if ((st = eltwise_check(op, n_inputs, need_x ? inputs : nullptr, top_diff, need_x))) return st;
    if (coeffs && op != CAFFE_ELTWISE_SUM) return fail(CAFFE_E_PARAM, "coefficients apply to SUM only");
    if (!bottom_diffs) return fail(CAFFE_E_INVALID, "bottom_diffs is NULL");
    for (int i = 0; i < n_inputs; i++) {
        if ((st = check_blob(bottom_diffs[i], "bottom_diff"))) return st;
        if ((st = same_elementwise(bottom_diffs[i], top_diff, "bottom_diffs and top_diff"))) return st;
        if (!aligned16(bottom_diffs[i]->ptr)) return fail(CAFFE_E_ALIGN, "bottom_diff %d must be 16-byte aligned", i);
        if (overlap(bottom_diffs[i], top_diff)) return fail(CAFFE_E_ALIAS, "bottom_diff %d overlaps top_diff", i);
        for (int j = 0; j < n_inputs; j++) {
            if (need_x && overlap(bottom_diffs[i], inputs[j])) return fail(CAFFE_E_ALIAS, "bottom_diff %d overlaps input %d", i, j);
            if (j != i && overlap(bottom_diffs[i], bottom_diffs[j])) return fail(CAFFE_E_ALIAS, "bottom_diffs %d and %d overlap", i, j);
        }
    }
    if (cnt(top_diff->shape) == 0) return CAFFE_OK;
    if (!aligned16(top_diff->ptr)) return fail(CAFFE_E_ALIGN, "top_diff must be 16-byte aligned");
    const void* in[CAFFE_ELTWISE_MAX_INPUTS];
    void* out[CAFFE_ELTWISE_MAX_INPUTS];
    for (int i = 0; i < n_inputs; i++) {
        in[i] = need_x ? inputs[i]->ptr : nullptr;
        out[i] = bottom_diffs[i]->ptr;
    }
    CK(eltwise_bwd_k(op, n_inputs, need_x ? in : nullptr, coeffs, top_diff->ptr, out, isbf(top_diff),
                     cnt(top_diff->shape), (cudaStream_t)stream),
       "eltwise bwd");
    return CAFFE_OK;
}

caffe_status caffe_hinge_loss(const caffe_blob* scores, const int32_t* labels, float* loss, caffe_blob* score_diff,
                              caffe_stream_t stream) {
    caffe_status st;
    if ((st = check_blob(scores, "scores"))) return st;
    if (!labels || !loss) return fail(CAFFE_E_INVALID, "labels and loss are required");
    const int N = scores->shape.n;
    const long long K = (long long)scores->shape.c * scores->shape.h * scores->shape.w;
    if (scores->shape.h * scores->shape.w != 1 && nhwc(scores)) return fail(CAFFE_E_INVALID, "scores must be (N,K,1,1) or NCHW");
    if (score_diff) {
        if ((st = check_blob(score_diff, "score_diff"))) return st;
        if (!same_shape(score_diff->shape, scores->shape)) return fail(CAFFE_E_SHAPE, "score_diff must match scores");
        if (score_diff->shape.h * score_diff->shape.w != 1 && nhwc(score_diff))
            return fail(CAFFE_E_INVALID, "score_diff must be NCHW");
        if (overlap(score_diff, scores)) return fail(CAFFE_E_ALIAS, "score_diff overlaps scores");
    }
    if (N == 0) return CAFFE_OK;
    CK(hinge_loss_k(scores->ptr, isbf(scores), labels, loss, score_diff ? score_diff->ptr : nullptr,
                    score_diff ? isbf(score_diff) : 0, N, (int)K, (cudaStream_t)stream),
       "hinge loss");
    return CAFFE_OK;
}

// ------------------------------------------------------------------ solver
static caffe_status lr_policy_check(const caffe_lr_policy* p) {
    if (!p) return fail(CAFFE_E_INVALID, "policy is NULL");
    if (p->policy != CAFFE_LR_FIXED && p->policy != CAFFE_LR_STEP && p->policy != CAFFE_LR_INV)
        return fail(CAFFE_E_INVALID, "bad lr policy %d", p->policy);
    if (p->policy == CAFFE_LR_STEP && p->stepsize < 1) return fail(CAFFE_E_PARAM, "step policy needs stepsize >= 1");
    return CAFFE_OK;
}

caffe_status caffe_lr_at_iter(const caffe_lr_policy* policy, int64_t iter, float* lr) {
    caffe_status st;
    if ((st = lr_policy_check(policy))) return st;
    if (!lr) return fail(CAFFE_E_INVALID, "lr is NULL");
    if (iter < 0) return fail(CAFFE_E_PARAM, "iter must be >= 0 (S:513)");
    *lr = (float)lr_policy_host(*policy, iter);
    return CAFFE_OK;
}

caffe_status caffe_solver_begin(const caffe_lr_policy* policy, caffe_solver_state* state, const float* loss,
                                caffe_stream_t stream) {
    caffe_status st;
    if ((st = lr_policy_check(policy))) return st;
    if (!state) return fail(CAFFE_E_INVALID, "state is NULL");
    if (reinterpret_cast<uintptr_t>(state) & 7) return fail(CAFFE_E_ALIGN, "state must be 8-byte aligned");
    CK(solver_begin_k(*policy, state, loss, (cudaStream_t)stream), "solver begin");
    return CAFFE_OK;
}

caffe_status caffe_solver_end(caffe_solver_state* state, caffe_stream_t stream) {
    if (!state) return fail(CAFFE_E_INVALID, "state is NULL");
    if (reinterpret_cast<uintptr_t>(state) & 7) return fail(CAFFE_E_ALIGN, "state must be 8-byte aligned");
    CK(solver_end_k(state, (cudaStream_t)stream), "solver end");
    return CAFFE_OK;
}

caffe_status caffe_sgd_update_solver(float* w, const float* g, float* v, void* w_bf16, int64_t count,
                                     const caffe_solver_state* state, float momentum, float decay, float grad_scale,
                                     caffe_stream_t stream) {
    if (count < 0) return fail(CAFFE_E_SHAPE, "negative count");
    if (count == 0) return CAFFE_OK;
    if (!w || !g || !v || !state) return fail(CAFFE_E_INVALID, "w, g, v and state are required");
    if (!aligned16(w) || !aligned16(g) || !aligned16(v) || (reinterpret_cast<uintptr_t>(w_bf16) & 7))
        return fail(CAFFE_E_ALIGN, "SGD buffers must be 16-byte aligned (w_bf16 8-byte)");
    CK(sgd_solver_k(w, g, v, w_bf16, count, state, momentum, decay, grad_scale, (cudaStream_t)stream),
       "sgd update (solver)");
    return CAFFE_OK;
}

}  // extern "C"
