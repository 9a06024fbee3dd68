/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * definitions of what the Caffe convolution hot path computes.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant with paper_1408_5093_b200/csrc (the CUDA path); neither
 * side includes or links the other.
 *
 * Authority (reference = /root/reference, cited as P:n for PAPER.md, S:n for
 * SPEC.md lines):
 *   - layer contract "forward pass ... backward pass computes the gradients
 *     with respect to the parameters and to the inputs"  P:156 (Sec. 3.2)
 *   - layer catalogue (convolution, pooling, inner products, ReLU, LRN,
 *     softmax loss)                                           P:158 (Sec. 3.2)
 *   - blob layout NCHW, index ((n*C+c)*H+h)*W+w
 *   - conv forward formula, zero padding, floor output size
 *   - conv backward, exact analytic gradients
 *   - grouped convolution: DESIGN.md reading R3
 *   - pooling formulas S:163; output size S:126 with reading R5;
 *     avg divisor reading R6; max tie/index reading R7; max backward order R8
 *   - LRN formula S:217 with alpha/n scaling and clipped window S:296 (R9)
 *   - im2col lowering S:297 / S:806 (col2im = its adjoint, fixed order, R8-style)
 *
 * Floating point: every accumulation is done in double (fp64) unless the
 * function name ends in _f32, in which case the paper-reading fixes an FP32
 * summation order so that a GPU kernel can be compared bit-exactly (R8).
 * Loops are the literal definitions: no blocking, no reordering, no fusion.
 * OpenMP only distributes independent outputs across threads; each output's
 * own summation order is the one written in the loop.
 *
 * Parity pins: see tests/test_oracle_*.py (SPEC worked examples, hand
 * brute-force cases, adjoint identities, independent im2col+matmul, finite
 * differences, FP64 torch.nn.functional cross-checks).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <float.h>

#define IDX4(n, c, h, w, C, H, W) ((((int64_t)(n) * (C) + (c)) * (H) + (h)) * (W) + (w))

/* output_h = (in_h + 2 pad_h - kernel_h)/stride_h + 1, floor division. */
int oracle_conv_out_dim(int in, int k, int s, int p) {
    int span = in + 2 * p - k;
    if (span < 0 || s < 1) return -1;
    return span / s + 1;
}

/*
 * Conv forward, S:145 with groups (R3):
 *   Y[n,o,y,x] = b[o] + sum_{c'<C/g, i<kh, j<kw} W[o,c',i,j] * X[n, (o/(O/g))*(C/g)+c', y*sh-ph+i, x*sw-pw+j]
 * out-of-range input positions contribute 0 (zero padding).
 * relu != 0 applies max(acc, 0) (fused ReLU).
 */
void oracle_conv_forward(const double* X, const double* Wt, const double* b,
                         int N, int C, int H, int W, int O, int kh, int kw,
                         int sh, int sw, int ph, int pw, int g, int relu, double* Y) {
    int OH = oracle_conv_out_dim(H, kh, sh, ph), OW = oracle_conv_out_dim(W, kw, sw, pw);
    int Cg = C / g, Og = O / g;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int o = 0; o < O; o++) {
            int cbase = (o / Og) * Cg;
            for (int y = 0; y < OH; y++)
                for (int x = 0; x < OW; x++) {
                    double acc = b ? b[o] : 0.0;
                    for (int c = 0; c < Cg; c++)
                        for (int i = 0; i < kh; i++)
                            for (int j = 0; j < kw; j++) {
                                int h = y * sh - ph + i, w = x * sw - pw + j;
                                if (h >= 0 && h < H && w >= 0 && w < W)
                                    acc += Wt[IDX4(o, c, i, j, Cg, kh, kw)] *
                                           X[IDX4(n, cbase + c, h, w, C, H, W)];
                            }
                    if (relu && !(acc > 0.0)) acc = 0.0;
                    Y[IDX4(n, o, y, x, O, OH, OW)] = acc;
                }
        }
}

/*
 * Conv backward w.r.t. data (exact adjoint of the forward map).
 * Scatter form of the same seven loops into a zeroed per-image sum G:
 *   G[n, g(o)C/g+c', y*sh-ph+i, x*sw-pw+j] += W[o,c',i,j] * dY[n,o,y,x];  dX = beta*dX + G
 * Parallel over n only (each image's dX is written by one thread, so the
 * summation order per element is the loop order o, y, x, c', i, j).
 */
void oracle_conv_backward_data(const double* dY, const double* Wt,
                               int N, int C, int H, int W, int O, int kh, int kw,
                               int sh, int sw, int ph, int pw, int g, double beta, double* dX) {
    int OH = oracle_conv_out_dim(H, kh, sh, ph), OW = oracle_conv_out_dim(W, kw, sw, pw);
    int Cg = C / g, Og = O / g;
#pragma omp parallel for schedule(static)
    for (int n = 0; n < N; n++) {
        /* the image's gradient is summed into a zeroed buffer, then dX = beta*dX + sum,
           so that beta=1 twice gives exactly 2x */
        double* acc = (double*)calloc((size_t)C * H * W, sizeof(double));
        for (int o = 0; o < O; o++) {
            int cbase = (o / Og) * Cg;
            for (int y = 0; y < OH; y++)
                for (int x = 0; x < OW; x++) {
                    double d = dY[IDX4(n, o, y, x, O, OH, OW)];
                    for (int c = 0; c < Cg; c++)
                        for (int i = 0; i < kh; i++)
                            for (int j = 0; j < kw; j++) {
                                int h = y * sh - ph + i, w = x * sw - pw + j;
                                if (h >= 0 && h < H && w >= 0 && w < W)
                                    acc[IDX4(0, cbase + c, h, w, C, H, W)] +=
                                        Wt[IDX4(o, c, i, j, Cg, kh, kw)] * d;
                            }
                }
        }
        for (int64_t e = 0; e < (int64_t)C * H * W; e++) {
            double* p = &dX[(int64_t)n * C * H * W + e];
            *p = (beta == 0.0 ? 0.0 : beta * *p) + acc[e];
        }
        free(acc);
    }
}

/*
 * Conv backward w.r.t. weights and bias (accumulate semantics via beta, R4):
 *   dW[o,c',i,j] = beta*dW + sum_{n,y,x} dY[n,o,y,x] * X[n, g(o)C/g+c', y*sh-ph+i, x*sw-pw+j]
 *   db[o]        = beta*db + sum_{n,y,x} dY[n,o,y,x]
 * Parallel over o (each filter's gradient is owned by one thread).
 */
void oracle_conv_backward_weight(const double* X, const double* dY,
                                 int N, int C, int H, int W, int O, int kh, int kw,
                                 int sh, int sw, int ph, int pw, int g, double beta,
                                 double* dW, double* db) {
    int OH = oracle_conv_out_dim(H, kh, sh, ph), OW = oracle_conv_out_dim(W, kw, sw, pw);
    int Cg = C / g, Og = O / g;
#pragma omp parallel for schedule(static)
    for (int o = 0; o < O; o++) {
        int cbase = (o / Og) * Cg;
        for (int c = 0; c < Cg; c++)
            for (int i = 0; i < kh; i++)
                for (int j = 0; j < kw; j++) {
                    double acc = 0.0;
                    for (int n = 0; n < N; n++)
                        for (int y = 0; y < OH; y++)
                            for (int x = 0; x < OW; x++) {
                                int h = y * sh - ph + i, w = x * sw - pw + j;
                                if (h >= 0 && h < H && w >= 0 && w < W)
                                    acc += dY[IDX4(n, o, y, x, O, OH, OW)] *
                                           X[IDX4(n, cbase + c, h, w, C, H, W)];
                            }
                    double* p = &dW[IDX4(o, c, i, j, Cg, kh, kw)];
                    *p = (beta == 0.0 ? 0.0 : beta * *p) + acc;
                }
        if (db) {
            double acc = 0.0;
            for (int n = 0; n < N; n++)
                for (int y = 0; y < OH; y++)
                    for (int x = 0; x < OW; x++) acc += dY[IDX4(n, o, y, x, O, OH, OW)];
            db[o] = (beta == 0.0 ? 0.0 : beta * db[o]) + acc;
        }
    }
}

/*
 * im2col for one image n ("explicit patch-matrix lowering"):
 *   col[(c*kh+i)*kw+j, y*OW+x] = X[n,c,y*sh-ph+i,x*sw-pw+j]  (0 if out of range)
 * Pure data movement -> bit-exact.
 */
void oracle_im2col_f32(const float* X, int n, int C, int H, int W, int kh, int kw,
                       int sh, int sw, int ph, int pw, float* col) {
    int OH = oracle_conv_out_dim(H, kh, sh, ph), OW = oracle_conv_out_dim(W, kw, sw, pw);
    for (int c = 0; c < C; c++)
        for (int i = 0; i < kh; i++)
            for (int j = 0; j < kw; j++)
                for (int y = 0; y < OH; y++)
                    for (int x = 0; x < OW; x++) {
                        int h = y * sh - ph + i, w = x * sw - pw + j;
                        float v = (h >= 0 && h < H && w >= 0 && w < W) ? X[IDX4(n, c, h, w, C, H, W)] : 0.0f;
                        col[((int64_t)(c * kh + i) * kw + j) * OH * OW + y * OW + x] = v;
                    }
}

/*
 * col2im for one image n: adjoint of im2col, written as a gather so that the
 * FP32 summation order is fixed (reading R8-style, SURVEY Sec. 8(c) loop nest):
 *   for each (c,h,w): acc = 0.0f; for y asc, x asc with i=h+ph-y*sh in [0,kh),
 *   j=w+pw-x*sw in [0,kw): acc += col[(c*kh+i)*kw+j, y*OW+x]; dX[n,c,h,w] = acc
 */
void oracle_col2im_f32(const float* col, int n, int C, int H, int W, int kh, int kw,
                       int sh, int sw, int ph, int pw, float* dX) {
    int OH = oracle_conv_out_dim(H, kh, sh, ph), OW = oracle_conv_out_dim(W, kw, sw, pw);
    for (int c = 0; c < C; c++)
        for (int h = 0; h < H; h++)
            for (int w = 0; w < W; w++) {
                float acc = 0.0f;
                for (int y = 0; y < OH; y++)
                    for (int x = 0; x < OW; x++) {
                        int i = h + ph - y * sh, j = w + pw - x * sw;
                        if (i >= 0 && i < kh && j >= 0 && j < kw)
                            acc += col[((int64_t)(c * kh + i) * kw + j) * OH * OW + y * OW + x];
                    }
                dX[IDX4(n, c, h, w, C, H, W)] = acc;
            }
}

/*
 * Pool output size, S:126 ceil rule with reading R5 (PyTorch ceil_mode rule):
 *   OH = ceil((H + 2p - k)/s) + 1;  if (OH-1)*s >= H + p then OH -= 1.
 */
int oracle_pool_out_dim(int in, int k, int s, int p) {
    int span = in + 2 * p - k;
    if (span < 0 || s < 1 || k < 1) return -1;
    int o = (span + s - 1) / s + 1;
    if ((o - 1) * s >= in + p) o -= 1;
    return o;
}

/*
 * Max pool forward (ties R7): window rows hs=py*s-p .. min(hs+k,H)-1
 * clipped at 0; scan h ascending, w ascending; a candidate replaces the
 * current best only if strictly greater; the first in-image element seeds the
 * scan.  mask = h*W + w within the (n,c) plane.  Pure selection -> bit-exact.
 * Written once for float (_f32: the GPU parity form) and double (_f64: the
 * fp64 net oracle, oracle/net.py) -- selection does not round, so both give
 * the same argmax on the same values.
 */
#define MAXPOOL_FWD_BODY(T)                                                               \
    int OH = oracle_pool_out_dim(H, kh, sh, ph), OW = oracle_pool_out_dim(W, kw, sw, pw);   \
    _Pragma("omp parallel for collapse(2) schedule(static)")                              \
    for (int n = 0; n < N; n++)                                                           \
        for (int c = 0; c < C; c++)                                                       \
            for (int py = 0; py < OH; py++)                                               \
                for (int px = 0; px < OW; px++) {                                         \
                    int hs = py * sh - ph, ws = px * sw - pw;                             \
                    int he = hs + kh < H ? hs + kh : H, we = ws + kw < W ? ws + kw : W;   \
                    if (hs < 0) hs = 0;                                                   \
                    if (ws < 0) ws = 0;                                                   \
                    T best = 0;                                                           \
                    int32_t arg = -1;                                                     \
                    for (int h = hs; h < he; h++)                                         \
                        for (int w = ws; w < we; w++) {                                   \
                            T v = X[IDX4(n, c, h, w, C, H, W)];                           \
                            if (arg < 0 || v > best) { best = v; arg = h * W + w; }       \
                        }                                                                 \
                    Y[IDX4(n, c, py, px, C, OH, OW)] = best;                              \
                    if (mask) mask[IDX4(n, c, py, px, C, OH, OW)] = arg;                  \
                }

void oracle_maxpool_forward_f32(const float* X, int N, int C, int H, int W,
                                int kh, int kw, int sh, int sw, int ph, int pw,
                                float* Y, int32_t* mask) {
    MAXPOOL_FWD_BODY(float)
}

void oracle_maxpool_forward_f64(const double* X, int N, int C, int H, int W,
                                int kh, int kw, int sh, int sw, int ph, int pw,
                                double* Y, int32_t* mask) {
    MAXPOOL_FWD_BODY(double)
}

/*
 * Max pool backward ("routed to its recorded argmax ... accumulating on
 * overlap"), written as a gather with reading R8's fixed order:
 *   dX[n,c,h,w] = sum over (py asc, px asc) with mask[n,c,py,px]==h*W+w of dY[n,c,py,px]
 * Only the windows that can contain (h,w) are visited -- rows py with
 * py*s-p <= h < py*s-p+k, i.e. ceil((h+p-k+1)/s) <= py <= floor((h+p)/s), clipped
 * to [0,OH) (same for columns) -- in the same ascending order; the windows
 * skipped cannot hold h*W+w in their mask and would add nothing.
 * _f32 sums in float (the GPU's bit-exact order), _f64 in double (oracle/net.py).
 */
static int win_lo(int h, int k, int s, int p) {   /* smallest py with py*s-p+k > h */
    int t = h + p - k + 1;
    int q = t <= 0 ? 0 : (t + s - 1) / s;
    return q;
}
static int win_hi(int h, int s, int p, int O) {   /* largest py with py*s-p <= h, clipped */
    int q = (h + p) / s;
    return q < O - 1 ? q : O - 1;
}
#define MAXPOOL_BWD_BODY(T)                                                               \
    int OH = oracle_pool_out_dim(H, kh, sh, ph), OW = oracle_pool_out_dim(W, kw, sw, pw);   \
    _Pragma("omp parallel for collapse(2) schedule(static)")                              \
    for (int n = 0; n < N; n++)                                                           \
        for (int c = 0; c < C; c++)                                                       \
            for (int h = 0; h < H; h++)                                                   \
                for (int w = 0; w < W; w++) {                                             \
                    T acc = 0;                                                            \
                    int y0 = win_lo(h, kh, sh, ph), y1 = win_hi(h, sh, ph, OH);           \
                    int x0 = win_lo(w, kw, sw, pw), x1 = win_hi(w, sw, pw, OW);           \
                    for (int py = y0; py <= y1; py++)                                     \
                        for (int px = x0; px <= x1; px++) {                               \
                            int64_t t = IDX4(n, c, py, px, C, OH, OW);                    \
                            if (mask[t] == h * W + w) acc += dY[t];                       \
                        }                                                                 \
                    dX[IDX4(n, c, h, w, C, H, W)] = acc;                                  \
                }

void oracle_maxpool_backward_f32(const float* dY, const int32_t* mask, int N, int C, int H, int W,
                                 int kh, int kw, int sh, int sw, int ph, int pw, float* dX) {
    MAXPOOL_BWD_BODY(float)
}

void oracle_maxpool_backward_f64(const double* dY, const int32_t* mask, int N, int C, int H, int W,
                                 int kh, int kw, int sh, int sw, int ph, int pw, double* dX) {
    MAXPOOL_BWD_BODY(double)
}

/*
 * Average pool forward (S:163 mean over the window; divisor reading R6):
 *   hs=py*s-p; he=min(hs+k, H+p); size=(he-hs)*(we-ws); clip to the image; Y = sum/size
 */
void oracle_avepool_forward(const double* X, int N, int C, int H, int W,
                            int kh, int kw, int sh, int sw, int ph, int pw, double* Y) {
    int OH = oracle_pool_out_dim(H, kh, sh, ph), OW = oracle_pool_out_dim(W, kw, sw, pw);
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++)
            for (int py = 0; py < OH; py++)
                for (int px = 0; px < OW; px++) {
                    int hs = py * sh - ph, ws = px * sw - pw;
                    int he = hs + kh < H + ph ? hs + kh : H + ph;
                    int we = ws + kw < W + pw ? ws + kw : W + pw;
                    int size = (he - hs) * (we - ws);
                    if (hs < 0) hs = 0;
                    if (ws < 0) ws = 0;
                    if (he > H) he = H;
                    if (we > W) we = W;
                    double acc = 0.0;
                    for (int h = hs; h < he; h++)
                        for (int w = ws; w < we; w++) acc += X[IDX4(n, c, h, w, C, H, W)];
                    Y[IDX4(n, c, py, px, C, OH, OW)] = acc / size;
                }
}

/* Average pool backward ("spread uniformly"): exact adjoint of the forward, scatter form. */
void oracle_avepool_backward(const double* dY, int N, int C, int H, int W,
                             int kh, int kw, int sh, int sw, int ph, int pw, double* dX) {
    int OH = oracle_pool_out_dim(H, kh, sh, ph), OW = oracle_pool_out_dim(W, kw, sw, pw);
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++) {
            for (int h = 0; h < H; h++)
                for (int w = 0; w < W; w++) dX[IDX4(n, c, h, w, C, H, W)] = 0.0;
            for (int py = 0; py < OH; py++)
                for (int px = 0; px < OW; px++) {
                    int hs = py * sh - ph, ws = px * sw - pw;
                    int he = hs + kh < H + ph ? hs + kh : H + ph;
                    int we = ws + kw < W + pw ? ws + kw : W + pw;
                    int size = (he - hs) * (we - ws);
                    if (hs < 0) hs = 0;
                    if (ws < 0) ws = 0;
                    if (he > H) he = H;
                    if (we > W) we = W;
                    double d = dY[IDX4(n, c, py, px, C, OH, OW)] / size;
                    for (int h = hs; h < he; h++)
                        for (int w = ws; w < we; w++) dX[IDX4(n, c, h, w, C, H, W)] += d;
                }
        }
}

/*
 * LRN across channels (reading R9):
 *   S[c] = k + alpha/n * sum_{c'=max(0,c-r)}^{min(C-1,c+r)} X[c']^2,  r=(n-1)/2
 *   Y[c] = X[c] * S[c]^(-beta)
 * scale (nullable) receives S.
 */
void oracle_lrn_forward(const double* X, int N, int C, int H, int W, int size,
                        double alpha, double beta, double k, double* Y, double* scale) {
    int r = (size - 1) / 2;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++)
            for (int h = 0; h < H; h++)
                for (int w = 0; w < W; w++) {
                    double s = 0.0;
                    int lo = c - r < 0 ? 0 : c - r, hi = c + r > C - 1 ? C - 1 : c + r;
                    for (int cc = lo; cc <= hi; cc++) {
                        double v = X[IDX4(n, cc, h, w, C, H, W)];
                        s += v * v;
                    }
                    double S = k + alpha / size * s;
                    int64_t t = IDX4(n, c, h, w, C, H, W);
                    Y[t] = X[t] * pow(S, -beta);
                    if (scale) scale[t] = S;
                }
}

/*
 * LRN backward: exact derivative of the forward map ("exact analytic
 * gradient").  With S_c as above and Y_c = X_c S_c^-beta,
 *   dX[c] = dY[c] * S_c^-beta - (2 alpha beta / n) * X[c] * sum_{c': c in win(c')} dY[c'] Y[c'] / S_c'
 * and c in win(c') <=> c' in win(c) (the window is symmetric and clipped).
 */
void oracle_lrn_backward(const double* X, const double* dY, int N, int C, int H, int W,
                         int size, double alpha, double beta, double k, double* dX) {
    int r = (size - 1) / 2;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++)
            for (int h = 0; h < H; h++)
                for (int w = 0; w < W; w++) {
                    double Sc = 0.0;
                    {
                        int lo = c - r < 0 ? 0 : c - r, hi = c + r > C - 1 ? C - 1 : c + r;
                        for (int cc = lo; cc <= hi; cc++) {
                            double v = X[IDX4(n, cc, h, w, C, H, W)];
                            Sc += v * v;
                        }
                        Sc = k + alpha / size * Sc;
                    }
                    double acc = 0.0;
                    int lo = c - r < 0 ? 0 : c - r, hi = c + r > C - 1 ? C - 1 : c + r;
                    for (int cp = lo; cp <= hi; cp++) {
                        double S = 0.0;
                        int lo2 = cp - r < 0 ? 0 : cp - r, hi2 = cp + r > C - 1 ? C - 1 : cp + r;
                        for (int cc = lo2; cc <= hi2; cc++) {
                            double v = X[IDX4(n, cc, h, w, C, H, W)];
                            S += v * v;
                        }
                        S = k + alpha / size * S;
                        int64_t t = IDX4(n, cp, h, w, C, H, W);
                        double Yp = X[t] * pow(S, -beta);
                        acc += dY[t] * Yp / S;
                    }
                    int64_t t = IDX4(n, c, h, w, C, H, W);
                    dX[t] = dY[t] * pow(Sc, -beta) - 2.0 * alpha * beta / size * X[t] * acc;
                }
}
