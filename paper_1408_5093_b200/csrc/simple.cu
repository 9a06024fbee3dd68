// simple.cu -- CUDA-core kernels: the FP32-FMA reference convolution (math mode CAFFE_MATH_FP32),
// im2col/col2im test entry points, and the bandwidth-bound neighbour layers (ReLU, max/avg pooling,
// LRN), softmax-with-loss, bias gradient and the SGD update.
// Formulas: conv S:145/S:154, pool S:163/S:172 (+R5..R8), LRN S:217/S:226 (R9), ReLU S:199/S:208,
// softmax loss S:253/S:262, SGD S:523 (R18).
//
// Every activation kernel is layout-generic: element (n,c,h,w) lives at n*sn + c*sc + h*sh + w*sw
// (L4), and threads walk the OUTPUT in its memory order so warps read/write consecutive addresses
// in either NCHW or NHWC.  Index math is 32-bit (blobs < 2^31 elements, checked by the ABI).
#include "internal.h"
#include "ptx.cuh"
#include <algorithm>

#include <cuda_bf16.h>
#include <cooperative_groups.h>

namespace cb {

__device__ __forceinline__ float ldv(const void* p, int i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void stv(void* p, int i, int bf16, float v) {
    if (bf16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(p)[i] = v;
}
static inline unsigned nblk(long long n, int t) {
    long long b = (n + t - 1) / t;
    if (b > 148LL * 32) b = 148LL * 32;
    return (unsigned)(b < 1 ? 1 : b);
}
#define GRID_STRIDE(t, total) \
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < (total); t += gridDim.x * blockDim.x)

// decode a linear index t of a (N,C,H,W) tensor stored with layout `nhwc` into (n,c,h,w)
__device__ __forceinline__ void decode(int t, int C, int H, int W, bool nhwc, int& n, int& c, int& h, int& w) {
    if (nhwc) {
        c = t % C; t /= C;
        w = t % W; t /= W;
        h = t % H; n = t / H;
    } else {
        w = t % W; t /= W;
        h = t % H; t /= H;
        c = t % C; n = t / C;
    }
}

__device__ __forceinline__ float tf32_round(float x) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// ================================================================ FP32 reference convolution
__global__ void conv_fwd_fp32_kernel(const void* __restrict__ x, int xb, L4 lx, const void* __restrict__ w, int wb,
                                     const float* __restrict__ b, void* __restrict__ y, int yb, L4 ly, int ynhwc,
                                     int relu, ConvGeom g, int total) {
    const int Cg = g.C / g.G, Og = g.O / g.G;
    GRID_STRIDE(t, total) {
        int n, o, oy, ox;
        decode(t, g.O, g.OH, g.OW, ynhwc, n, o, oy, ox);
        const int cb = (o / Og) * Cg;
        float acc = 0.f;
        for (int c = 0; c < Cg; c++)
            for (int i = 0; i < g.kh; i++) {
                const int h = oy * g.sh - g.ph + i;
                if (h < 0 || h >= g.H) continue;
                for (int j = 0; j < g.kw; j++) {
                    const int ww = ox * g.sw - g.pw + j;
                    if (ww < 0 || ww >= g.W) continue;
                    acc = fmaf(ldv(w, ((o * Cg + c) * g.kh + i) * g.kw + j, wb),
                               ldv(x, n * lx.sn + (cb + c) * lx.sc + h * lx.sh + ww * lx.sw, xb), acc);
                }
            }
        if (b) acc += b[o];
        if (relu && !(acc > 0.f)) acc = 0.f;
        stv(y, t, yb, acc);
    }
}

cudaError_t fp32_conv_fwd(const void* x, int x_bf16, L4 lx, const void* w, int w_bf16, const float* b, void* y,
                          int y_bf16, L4 ly, int ynhwc, int relu, const ConvGeom& g, cudaStream_t s) {
    const int total = g.N * g.O * g.OH * g.OW;
    conv_fwd_fp32_kernel<<<nblk(total, 256), 256, 0, s>>>(x, x_bf16, lx, w, w_bf16, b, y, y_bf16, ly, ynhwc, relu, g,
                                                           total);
    note_launch();
    return cudaGetLastError();
}

// gather form of the data gradient: dX[n,c,h,w] = sum_{o in grp(c), i, j : y=(h+ph-i)/sh, x=(w+pw-j)/sw integral}
__global__ void conv_dgrad_fp32_kernel(const void* __restrict__ dy, int dyb, L4 ly, const void* __restrict__ w, int wb,
                                       void* __restrict__ dx, int dxb, int xnhwc, float beta, ConvGeom g, int total,
                                       int tf32) {
    const int Cg = g.C / g.G, Og = g.O / g.G;
    GRID_STRIDE(t, total) {
        int n, c, h, ww;
        decode(t, g.C, g.H, g.W, xnhwc, n, c, h, ww);
        const int grp = c / Cg, cl = c % Cg;
        float acc = 0.f;
        for (int o = grp * Og; o < (grp + 1) * Og; o++)
            for (int i = 0; i < g.kh; i++) {
                const int yy = h + g.ph - i;
                if (yy < 0 || yy % g.sh) continue;
                const int oy = yy / g.sh;
                if (oy >= g.OH) continue;
                for (int j = 0; j < g.kw; j++) {
                    const int xx = ww + g.pw - j;
                    if (xx < 0 || xx % g.sw) continue;
                    const int ox = xx / g.sw;
                    if (ox >= g.OW) continue;
                    float a = ldv(w, ((o * Cg + cl) * g.kh + i) * g.kw + j, wb);
                    float d = ldv(dy, n * ly.sn + o * ly.sc + oy * ly.sh + ox * ly.sw, dyb);
                    if (tf32) { a = tf32_round(a); d = tf32_round(d); }
                    acc = fmaf(a, d, acc);
                }
            }
        if (beta != 0.f) acc += beta * ldv(dx, t, dxb);
        stv(dx, t, dxb, acc);
    }
}

cudaError_t fp32_conv_dgrad(const void* dy, int dy_bf16, L4 ly, const void* w, int w_bf16, void* dx, int dx_bf16,
                            int xnhwc, float beta, const ConvGeom& g, cudaStream_t s, int tf32) {
    const int total = g.N * g.C * g.H * g.W;
    conv_dgrad_fp32_kernel<<<nblk(total, 256), 256, 0, s>>>(dy, dy_bf16, ly, w, w_bf16, dx, dx_bf16, xnhwc, beta, g,
                                                             total, tf32);
    note_launch();
    return cudaGetLastError();
}

// Block per weight element; each thread sums a fixed strided subset of the (n, y, x) range, then a
// fixed-shape tree reduction -> deterministic, blocked FP32 summation (reading R13).
__global__ void conv_wgrad_fp32_kernel(const void* __restrict__ x, int xb, L4 lx, const void* __restrict__ dy, int dyb,
                                       L4 ly, float* __restrict__ dw, float beta, ConvGeom g, int tf32) {
    __shared__ float red[256];
    const int Cg = g.C / g.G, Og = g.O / g.G;
    const int widx = blockIdx.x;
    const int j = widx % g.kw;
    int r = widx / g.kw;
    const int i = r % g.kh;
    r /= g.kh;
    const int c = r % Cg;
    const int o = r / Cg;
    const int cfull = (o / Og) * Cg + c;
    const int P = g.OH * g.OW, tot = g.N * P;
    float acc = 0.f;
    for (int q = threadIdx.x; q < tot; q += blockDim.x) {
        const int n = q / P;
        const int p = q - n * P;
        const int oy = p / g.OW, ox = p - oy * g.OW;
        const int h = oy * g.sh - g.ph + i, ww = ox * g.sw - g.pw + j;
        if (h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
        float d = ldv(dy, n * ly.sn + o * ly.sc + oy * ly.sh + ox * ly.sw, dyb);
        float v = ldv(x, n * lx.sn + cfull * lx.sc + h * lx.sh + ww * lx.sw, xb);
        if (tf32) { d = tf32_round(d); v = tf32_round(v); }
        acc = fmaf(d, v, acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) dw[widx] = (beta != 0.f ? beta * dw[widx] : 0.f) + red[0];
}

cudaError_t fp32_conv_wgrad(const void* x, int x_bf16, L4 lx, const void* dy, int dy_bf16, L4 ly, float* dw,
                            float beta, const ConvGeom& g, cudaStream_t s, int tf32) {
    const int nw = g.O * (g.C / g.G) * g.kh * g.kw;
    conv_wgrad_fp32_kernel<<<(unsigned)nw, 256, 0, s>>>(x, x_bf16, lx, dy, dy_bf16, ly, dw, beta, g, tf32);
    note_launch();
    return cudaGetLastError();
}

// ================================================================ bias gradient (deterministic, 2 stages)
// db[o] = beta*db + sum_{n,p} dY[n,o,p].  Stage 1: partial[s][o] over a fixed pixel range s.
//   NHWC (channels contiguous): lane -> channel, 8 warps stride over the pixels of the range.
//   NCHW (pixels contiguous):   block = (range, channel), threads stride over the range.
// Stage 2: sum of the partials in ascending s.
constexpr int BG_SPLITS_MAX = 148 * 8;

__global__ void bias_partial_nhwc(const void* __restrict__ dy, int dyb, int O, int M, int R, float* __restrict__ part) {
    __shared__ float red[8][33];
    const int s = blockIdx.x, c = blockIdx.y * 32 + (threadIdx.x & 31), wp = threadIdx.x >> 5;
    float acc = 0.f;
    if (c < O) {
        const int m1 = min(M, (s + 1) * R);
        for (int m = s * R + wp; m < m1; m += 8) acc += ldv(dy, m * O + c, dyb);
    }
    red[wp][threadIdx.x & 31] = acc;
    __syncthreads();
    if (wp == 0 && c < O) {
        float t = 0.f;
        for (int k = 0; k < 8; k++) t += red[k][threadIdx.x];
        part[s * O + c] = t;
    }
}

// BF16 channels-last, O % 8 == 0: thread = (row group, 8-channel vector); 16-byte loads; the row
// groups of a block are summed in fixed order through shared memory.
__global__ void bias_partial_nhwc8(const __nv_bfloat16* __restrict__ dy, int O, int M, int R, float* __restrict__ part) {
    extern __shared__ float red8[];   // [RG][O]
    const int CV = O / 8, RG = blockDim.x / CV;
    const int s = blockIdx.x, cv = threadIdx.x % CV, rg = threadIdx.x / CV;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; e++) acc[e] = 0.f;
    if (rg < RG) {
        const int m1 = min(M, (s + 1) * R);
#pragma unroll 4
        for (int m = s * R + rg; m < m1; m += RG) {
            const uint4 u = *reinterpret_cast<const uint4*>(dy + (long long)m * O + cv * 8);
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const float2 f = __bfloat1622float2(h[e]);
                acc[2 * e] += f.x;
                acc[2 * e + 1] += f.y;
            }
        }
#pragma unroll
        for (int e = 0; e < 8; e++) red8[rg * O + cv * 8 + e] = acc[e];
    }
    __syncthreads();
    for (int o = threadIdx.x; o < O; o += blockDim.x) {
        float t = 0.f;
        for (int k = 0; k < RG; k++) t += red8[k * O + o];
        part[s * O + o] = t;
    }
}

__global__ void bias_partial_nchw(const void* __restrict__ dy, int dyb, int O, int P, int N, int R,
                                  float* __restrict__ part) {
    __shared__ float red[256];
    const int s = blockIdx.x, o = blockIdx.y;
    const int M = N * P, m1 = min(M, (s + 1) * R);
    float acc = 0.f;
    for (int m = s * R + threadIdx.x; m < m1; m += blockDim.x) {
        const int n = m / P, p = m - n * P;
        acc += ldv(dy, (n * O + o) * P + p, dyb);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[s * O + o] = red[0];
}

// Stage 2: block per output channel; threads take partials s = t, t+128, ... then a fixed tree.
__global__ void bias_final(const float* __restrict__ part, int S, int O, float* __restrict__ db, float beta) {
    __shared__ float red[128];
    const int o = blockIdx.x;
    float t = 0.f;
    for (int s = threadIdx.x; s < S; s += 128) t += part[s * O + o];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int st = 64; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) db[o] = (beta != 0.f ? beta * db[o] : 0.f) + red[0];
}

// splits of the pixel range: ~8 blocks per SM, >= 64 rows each
int g_bias_split_rows = 64;   // CAFFE_TUNE_BIAS_SPLIT_ROWS: rows per bias-gradient split (8 .. 1024)
int bias_grad_splits(int N, int O, int P) {
    const long long M = (long long)N * P;
    long long S = (M + g_bias_split_rows - 1) / g_bias_split_rows;
    if (S > BG_SPLITS_MAX) S = BG_SPLITS_MAX;
    return S < 1 ? 1 : (int)S;
}

// One pass for short reductions (an inner product's bias: M = batch rows of O columns): block = 32
// columns x 8 warps; warp w sums rows w, w+8, ... in ascending order (8 loads in flight), then the
// 8 warp sums are added in warp order -- deterministic, one launch instead of partials + final
// (which took 4096 blocks for fc6/fc7).
__global__ void __launch_bounds__(256) bias_rows_kernel(const void* __restrict__ dy, int dyb, int O, int M,
                                                        float* __restrict__ db, float beta) {
    __shared__ float red[8][33];
    const int c = blockIdx.x * 32 + (threadIdx.x & 31), wp = threadIdx.x >> 5;
    float acc = 0.f;
    if (c < O) {
        int m = wp;
        for (; m + 56 < M; m += 64) {
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = ldv(dy, (long long)(m + 8 * k) * O + c, dyb);
#pragma unroll
            for (int k = 0; k < 8; k++) acc += v[k];
        }
        for (; m < M; m += 8) acc += ldv(dy, (long long)m * O + c, dyb);
    }
    red[wp][threadIdx.x & 31] = acc;
    __syncthreads();
    if (wp == 0 && c < O) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; k++) t += red[k][threadIdx.x];
        db[c] = (beta != 0.f ? beta * db[c] : 0.f) + t;
    }
}
int g_bias_rows = 0;   // CAFFE_TUNE_BIAS_ROWS (measured slower in the step: 1.58-1.61 vs 1.47-1.52 ms)

cudaError_t bias_grad(const void* dy, int dy_bf16, int nhwc, float* db, float beta, int N, int O, int P, float* part,
                      cudaStream_t s) {
    const int M = N * P;
    if (g_bias_rows && P == 1 && M <= 8192) {
        bias_rows_kernel<<<(O + 31) / 32, 256, 0, s>>>(dy, dy_bf16, O, M, db, beta);
        note_launch();
        return cudaGetLastError();
    }
    const int S = bias_grad_splits(N, O, P);
    const int R = (M + S - 1) / S;
    if ((nhwc || P == 1) && dy_bf16 && O % 8 == 0 && O <= 2048 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0) {
        const int CV = O / 8, RG = 256 / CV;
        bias_partial_nhwc8<<<S, 256, (size_t)RG * O * sizeof(float), s>>>((const __nv_bfloat16*)dy, O, M, R, part);
    } else if (nhwc || P == 1) {
        bias_partial_nhwc<<<dim3(S, (O + 31) / 32), 256, 0, s>>>(dy, dy_bf16, O, M, R, part);
    } else {
        bias_partial_nchw<<<dim3(S, O), 256, 0, s>>>(dy, dy_bf16, O, P, N, R, part);
    }
    note_launch();
    bias_final<<<O, 128, 0, s>>>(part, S, O, db, beta);
    note_launch();
    return cudaGetLastError();
}

// ================================================================ im2col / col2im (bit-exact test entry points)
__global__ void im2col_kernel(const float* __restrict__ x, int n, ConvGeom g, float* __restrict__ col, int total) {
    const int P = g.OH * g.OW;
    GRID_STRIDE(t, total) {
        const int p = t % P, row = t / P;
        const int j = row % g.kw;
        const int i = (row / g.kw) % g.kh;
        const int c = row / (g.kw * g.kh);
        const int oy = p / g.OW, ox = p % g.OW;
        const int h = oy * g.sh - g.ph + i, w = ox * g.sw - g.pw + j;
        col[t] = (h >= 0 && h < g.H && w >= 0 && w < g.W) ? x[((n * g.C + c) * g.H + h) * g.W + w] : 0.f;
    }
}

cudaError_t im2col_k(const float* x, int n, const ConvGeom& g, float* col, cudaStream_t s) {
    const int total = g.C * g.kh * g.kw * g.OH * g.OW;
    im2col_kernel<<<nblk(total, 256), 256, 0, s>>>(x, n, g, col, total);
    note_launch();
    return cudaGetLastError();
}

// gather: for each (c,h,w) sum col over (y asc, x asc) -- the FP32 order fixed by the reading.
__global__ void col2im_kernel(const float* __restrict__ col, int n, ConvGeom g, float* __restrict__ dx, int total) {
    const int P = g.OH * g.OW;
    GRID_STRIDE(t, total) {
        const int w = t % g.W;
        const int h = (t / g.W) % g.H;
        const int c = t / (g.W * g.H);
        float acc = 0.f;
        for (int oy = 0; oy < g.OH; oy++) {
            const int i = h + g.ph - oy * g.sh;
            if (i < 0 || i >= g.kh) continue;
            for (int ox = 0; ox < g.OW; ox++) {
                const int j = w + g.pw - ox * g.sw;
                if (j < 0 || j >= g.kw) continue;
                acc += col[((c * g.kh + i) * g.kw + j) * P + oy * g.OW + ox];
            }
        }
        dx[n * g.C * g.H * g.W + t] = acc;
    }
}

cudaError_t col2im_k(const float* col, int n, const ConvGeom& g, float* dx, cudaStream_t s) {
    const int total = g.C * g.H * g.W;
    col2im_kernel<<<nblk(total, 256), 256, 0, s>>>(col, n, g, dx, total);
    note_launch();
    return cudaGetLastError();
}

// ================================================================ ReLU (vectorised, in-place safe)
__global__ void relu_fwd_f32(const float* __restrict__ x, float* y, int n) {
    const int n4 = n / 4;
    GRID_STRIDE(t, n4) {
        float4 v = reinterpret_cast<const float4*>(x)[t];
        v.x = v.x > 0.f ? v.x : 0.f; v.y = v.y > 0.f ? v.y : 0.f;
        v.z = v.z > 0.f ? v.z : 0.f; v.w = v.w > 0.f ? v.w : 0.f;
        reinterpret_cast<float4*>(y)[t] = v;
    }
    GRID_STRIDE(t, n - n4 * 4) { const float v = x[n4 * 4 + t]; y[n4 * 4 + t] = v > 0.f ? v : 0.f; }
}
__device__ __forceinline__ __nv_bfloat162 relu2(__nv_bfloat162 h) {
    const float2 f = __bfloat1622float2(h);
    return __floats2bfloat162_rn(f.x > 0.f ? f.x : 0.f, f.y > 0.f ? f.y : 0.f);
}
__global__ void relu_fwd_bf16(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* y, int n) {
    const int n8 = n / 8;
    GRID_STRIDE(t, n8) {
        uint4 v = reinterpret_cast<const uint4*>(x)[t];
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int e = 0; e < 4; e++) h[e] = relu2(h[e]);
        reinterpret_cast<uint4*>(y)[t] = v;
    }
    GRID_STRIDE(t, n - n8 * 8) {
        const float v = __bfloat162float(x[n8 * 8 + t]);
        y[n8 * 8 + t] = __float2bfloat16_rn(v > 0.f ? v : 0.f);
    }
}

cudaError_t relu_fwd(const void* x, void* y, int bf16, int count, cudaStream_t s) {
    if (bf16) relu_fwd_bf16<<<nblk(count / 8 + 1, 256), 256, 0, s>>>((const __nv_bfloat16*)x, (__nv_bfloat16*)y, count);
    else relu_fwd_f32<<<nblk(count / 4 + 1, 256), 256, 0, s>>>((const float*)x, (float*)y, count);
    note_launch();
    return cudaGetLastError();
}

// dx = x > 0 ? dy : 0 -- vectorised for bf16 x and bf16 dy (8 per thread), scalar otherwise.
__global__ void relu_bwd_bf16(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* dy, __nv_bfloat16* dx, int n) {
    const int n8 = n / 8;
    GRID_STRIDE(t, n8) {
        uint4 xv = reinterpret_cast<const uint4*>(x)[t];
        uint4 gv = reinterpret_cast<const uint4*>(dy)[t];
        const __nv_bfloat16* xh = reinterpret_cast<const __nv_bfloat16*>(&xv);
        __nv_bfloat16* gh = reinterpret_cast<__nv_bfloat16*>(&gv);
#pragma unroll
        for (int e = 0; e < 8; e++)
            if (!(__bfloat162float(xh[e]) > 0.f)) gh[e] = __float2bfloat16_rn(0.f);
        reinterpret_cast<uint4*>(dx)[t] = gv;
    }
    GRID_STRIDE(t, n - n8 * 8) {
        const int i = n8 * 8 + t;
        dx[i] = __bfloat162float(x[i]) > 0.f ? dy[i] : __float2bfloat16_rn(0.f);
    }
}
__global__ void relu_bwd_kernel(const void* __restrict__ x, const void* dy, void* dx, int xb, int db, int n) {
    GRID_STRIDE(t, n) {
        const float xv = ldv(x, t, xb);
        const float g = ldv(dy, t, db);
        stv(dx, t, db, xv > 0.f ? g : 0.f);
    }
}

cudaError_t relu_bwd(const void* x, const void* dy, void* dx, int x_bf16, int d_bf16, int count, cudaStream_t s) {
    const bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx)) & 15) == 0;
    if (x_bf16 && d_bf16 && al)
        relu_bwd_bf16<<<nblk(count / 8 + 1, 256), 256, 0, s>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)dy,
                                                               (__nv_bfloat16*)dx, count);
    else
        relu_bwd_kernel<<<nblk(count, 256), 256, 0, s>>>(x, dy, dx, x_bf16, d_bf16, count);
    note_launch();
    return cudaGetLastError();
}

// ================================================================ pooling
// Forward: thread per output element in the top's memory order.
__global__ void maxpool_fwd_kernel(const void* __restrict__ x, L4 lx, void* __restrict__ y, int ynhwc,
                                   void* __restrict__ mask, int mask_u8, int bf16, PoolGeom g, int total) {
    GRID_STRIDE(t, total) {
        int n, c, py, px;
        decode(t, g.C, g.OH, g.OW, ynhwc, n, c, py, px);
        const int hs0 = py * g.sh - g.ph, ws0 = px * g.sw - g.pw;
        const int he = min(hs0 + g.kh, g.H), we = min(ws0 + g.kw, g.W);
        const int hs = max(hs0, 0), ws = max(ws0, 0);
        const int base = n * lx.sn + c * lx.sc;
        float best = 0.f;
        int ah = -1, aw = 0;
        for (int h = hs; h < he; h++)
            for (int w = ws; w < we; w++) {
                const float v = ldv(x, base + h * lx.sh + w * lx.sw, bf16);
                if (ah < 0 || v > best) { best = v; ah = h; aw = w; }
            }
        stv(y, t, bf16, best);
        if (mask) {
            if (mask_u8) reinterpret_cast<uint8_t*>(mask)[t] = (uint8_t)((ah - hs0) * g.kw + (aw - ws0));
            else reinterpret_cast<int32_t*>(mask)[t] = ah * g.W + aw;
        }
    }
}

// ---- channels-last BF16 fast paths: one thread = one pixel x 8 consecutive channels (16-byte
// vectors), so every window access is a coalesced 16-byte load and index math is per pixel.
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const float2 t = __bfloat1622float2(h[e]);
        f[2 * e] = t.x;
        f[2 * e + 1] = t.y;
    }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; e++) h[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    return u;
}

// KH, KW > 0: compile-time window, fully unrolled so all of a thread's window loads are in flight
// at once (a runtime-bounded loop leaves one load outstanding per thread: latency-bound).
template <int KH, int KW>
__global__ void maxpool_fwd_nhwc8(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                  void* __restrict__ mask, int mask_u8, PoolGeom g, int total) {
    const int cv = g.C / 8;
    GRID_STRIDE(t, total) {
        const int c0 = (t % cv) * 8;
        int r = t / cv;
        const int px = r % g.OW; r /= g.OW;
        const int py = r % g.OH;
        const int n = r / g.OH;
        int hs = py * g.sh - g.ph, ws = px * g.sw - g.pw;
        const int hs0 = hs, ws0 = ws;   // unclipped window start (origin of a U8 window-local mask)
        const int he = min(hs + g.kh, g.H), we = min(ws + g.kw, g.W);
        hs = max(hs, 0);
        ws = max(ws, 0);
        float best[8];
        int arg[8];
#pragma unroll
        for (int e = 0; e < 8; e++) { best[e] = 0.f; arg[e] = -1; }
        if (KH > 0) {
            // Packed form of the strict '>' scan (R7): per bf16 pair, __hgt2_mask gives 0xFFFF lanes
            // where the new value is strictly greater (false for NaN, as in the scalar scan); the
            // running max and the running local window index (two 16-bit indices per word) are
            // updated with bit selects.  The first in-image element seeds (it is never clipped).
            uint4 raw[KH > 0 ? KH : 1][KW > 0 ? KW : 1];
#pragma unroll
            for (int i = 0; i < KH; i++)
#pragma unroll
                for (int j = 0; j < KW; j++)
                    if (hs + i < he && ws + j < we)
                        raw[i][j] = *reinterpret_cast<const uint4*>(
                            x + (((long long)n * g.H + hs + i) * g.W + ws + j) * g.C + c0);
            uint32_t bw[4] = {raw[0][0].x, raw[0][0].y, raw[0][0].z, raw[0][0].w};
            uint32_t aw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int i = 0; i < KH; i++)
#pragma unroll
                for (int j = 0; j < KW; j++) {
                    if (i == 0 && j == 0) continue;
                    if (hs + i < he && ws + j < we) {
                        const uint32_t vw[4] = {raw[i][j].x, raw[i][j].y, raw[i][j].z, raw[i][j].w};
                        const uint32_t pp = (uint32_t)(i * KW + j) * 0x00010001u;
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vw[e]),
                                                           *reinterpret_cast<const __nv_bfloat162*>(&bw[e]));
                            bw[e] = (vw[e] & m) | (bw[e] & ~m);
                            aw[e] = (pp & m) | (aw[e] & ~m);
                        }
                    }
                }
            const long long o = (long long)t * 8;
            *reinterpret_cast<uint4*>(y + o) = make_uint4(bw[0], bw[1], bw[2], bw[3]);
            if (mask) {
                if (mask_u8) {
                    // local index in the unclipped window: (hs - hs0 + i)*kw + (ws - ws0 + j)
                    const int shift = (hs - hs0) * g.kw + (ws - ws0);
                    uint32_t pk[2] = {0u, 0u};
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int p0 = (int)(aw[e] & 0xFFFFu), p1 = (int)(aw[e] >> 16);
                        const uint32_t l0 = (uint32_t)(shift + (p0 / KW) * g.kw + p0 % KW);
                        const uint32_t l1 = (uint32_t)(shift + (p1 / KW) * g.kw + p1 % KW);
                        pk[e >> 1] |= (l0 | (l1 << 8)) << (16 * (e & 1));
                    }
                    *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(mask) + o) = make_uint2(pk[0], pk[1]);
                } else {
                    int am[8];
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int p0 = (int)(aw[e] & 0xFFFFu), p1 = (int)(aw[e] >> 16);
                        am[2 * e] = (hs + p0 / KW) * g.W + ws + p0 % KW;
                        am[2 * e + 1] = (hs + p1 / KW) * g.W + ws + p1 % KW;
                    }
                    int4* mp = reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(mask) + o);
                    mp[0] = make_int4(am[0], am[1], am[2], am[3]);
                    mp[1] = make_int4(am[4], am[5], am[6], am[7]);
                }
            }
            continue;
        } else {
            for (int h = hs; h < he; h++)
                for (int w = ws; w < we; w++) {
                    float v[8];
                    unpack8(*reinterpret_cast<const uint4*>(x + (((long long)n * g.H + h) * g.W + w) * g.C + c0), v);
                    const int me = h * g.W + w;
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if (arg[e] < 0 || v[e] > best[e]) { best[e] = v[e]; arg[e] = me; }
                }
        }
        const long long o = (long long)t * 8;
        *reinterpret_cast<uint4*>(y + o) = pack8(best);
        if (mask) {
            if (mask_u8) {
                uint8_t* m = reinterpret_cast<uint8_t*>(mask) + o;
#pragma unroll
                for (int e = 0; e < 8; e++) m[e] = (uint8_t)((arg[e] / g.W - hs0) * g.kw + (arg[e] % g.W - ws0));
            } else {
                int4* m = reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(mask) + o);
                m[0] = make_int4(arg[0], arg[1], arg[2], arg[3]);
                m[1] = make_int4(arg[4], arg[5], arg[6], arg[7]);
            }
        }
    }
}

// Thread = one SH x SW block of input positions x 8 channels (SH, SW = the pool stride when it is
// 2x2, else 1x1).  Every window overlapping the block is loaded once -- mask, top_diff and, when
// fused, top -- and added to each block position it selected, in ascending (py, px) order, so each
// position's FP32 sum has R8's order (bit-exact); for 3x3/s2 windows this loads each window 4
// times instead of 9.  top != nullptr: fused backward of the ReLU that feeds the pool -- a window
// passes its gradient only when its max (= the ReLU output at the argmax) is > 0, which is exactly
// relu_bwd(pool_bwd(dy)).
// NPY x NPX (> 0): compile-time bound on the windows overlapping a block, so the window loads of
// a thread are unrolled and all in flight together.
template <int SH, int SW, int NPY, int NPX, bool MU8>
__global__ void maxpool_bwd_nhwc8(const __nv_bfloat16* __restrict__ dy, const void* __restrict__ mask,
                                  const __nv_bfloat16* __restrict__ top, __nv_bfloat16* __restrict__ dx, PoolGeom g,
                                  int HB, int WB, int total) {
    const int cv = g.C / 8;
    GRID_STRIDE(t, total) {
        const int c0 = (t % cv) * 8;
        int r = t / cv;
        const int bw = r % WB; r /= WB;
        const int bh = r % HB;
        const int n = r / HB;
        const int h0 = bh * SH, w0 = bw * SW;
        const int h1 = min(h0 + SH, g.H) - 1, w1 = min(w0 + SW, g.W) - 1;
        const int py0 = max(0, (h0 + g.ph - g.kh + g.sh) / g.sh), py1 = min(g.OH - 1, (h1 + g.ph) / g.sh);
        const int px0 = max(0, (w0 + g.pw - g.kw + g.sw) / g.sw), px1 = min(g.OW - 1, (w1 + g.pw) / g.sw);
        float acc[SH][SW][8];
#pragma unroll
        for (int i = 0; i < SH; i++)
#pragma unroll
            for (int j = 0; j < SW; j++)
#pragma unroll
                for (int e = 0; e < 8; e++) acc[i][j][e] = 0.f;
        // window (py, px): mask words (int32: 8 absolute indices; U8: 8 window-local bytes)
        auto window = [&](int py, int px, const int4& m0, const int4& m1, const uint2& mb, const uint4& dr,
                          const uint4& tr) {
            int mm[8];
            if (MU8) {
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    mm[e] = (int)((mb.x >> (8 * e)) & 0xffu);
                    mm[4 + e] = (int)((mb.y >> (8 * e)) & 0xffu);
                }
            } else {
                mm[0] = m0.x; mm[1] = m0.y; mm[2] = m0.z; mm[3] = m0.w;
                mm[4] = m1.x; mm[5] = m1.y; mm[6] = m1.z; mm[7] = m1.w;
            }
            float v[8];
            unpack8(dr, v);
            if (top) {
                float tv[8];
                unpack8(tr, tv);
#pragma unroll
                for (int e = 0; e < 8; e++)
                    if (!(tv[e] > 0.f)) v[e] = 0.f;
            }
            const int hs0 = py * g.sh - g.ph, ws0 = px * g.sw - g.pw;
#pragma unroll
            for (int i = 0; i < SH; i++)
#pragma unroll
                for (int j = 0; j < SW; j++) {
                    // U8: the block position's index local to this window, -1 when the position lies
                    // outside it (a local index would otherwise alias another row of the window)
                    const int li = h0 + i - hs0, lj = w0 + j - ws0;
                    const int me = MU8 ? ((li >= 0 && li < g.kh && lj >= 0 && lj < g.kw) ? li * g.kw + lj : -1)
                                       : (h0 + i) * g.W + (w0 + j);
#pragma unroll
                    for (int e = 0; e < 8; e++)
                        if (mm[e] == me) acc[i][j][e] += v[e];
                }
        };
        const int32_t* mask32 = reinterpret_cast<const int32_t*>(mask);
        const uint8_t* mask8 = reinterpret_cast<const uint8_t*>(mask);
        if (NPY > 0) {
            int4 m0[NPY > 0 ? NPY : 1][NPX > 0 ? NPX : 1], m1[NPY > 0 ? NPY : 1][NPX > 0 ? NPX : 1];
            uint2 mb[NPY > 0 ? NPY : 1][NPX > 0 ? NPX : 1];
            uint4 dr[NPY > 0 ? NPY : 1][NPX > 0 ? NPX : 1], tr[NPY > 0 ? NPY : 1][NPX > 0 ? NPX : 1];
#pragma unroll
            for (int a = 0; a < NPY; a++)
#pragma unroll
                for (int b = 0; b < NPX; b++)
                    if (py0 + a <= py1 && px0 + b <= px1) {
                        const long long q = (((long long)n * g.OH + py0 + a) * g.OW + px0 + b) * g.C + c0;
                        if (MU8) {
                            mb[a][b] = *reinterpret_cast<const uint2*>(mask8 + q);
                        } else {
                            m0[a][b] = *reinterpret_cast<const int4*>(mask32 + q);
                            m1[a][b] = *reinterpret_cast<const int4*>(mask32 + q + 4);
                        }
                        dr[a][b] = *reinterpret_cast<const uint4*>(dy + q);
                        if (top) tr[a][b] = *reinterpret_cast<const uint4*>(top + q);
                    }
#pragma unroll
            for (int a = 0; a < NPY; a++)
#pragma unroll
                for (int b = 0; b < NPX; b++)
                    if (py0 + a <= py1 && px0 + b <= px1)
                        window(py0 + a, px0 + b, m0[a][b], m1[a][b], mb[a][b], dr[a][b], tr[a][b]);
        } else {
            for (int py = py0; py <= py1; py++)
                for (int px = px0; px <= px1; px++) {
                    const long long q = (((long long)n * g.OH + py) * g.OW + px) * g.C + c0;
                    int4 a0 = make_int4(0, 0, 0, 0), a1 = make_int4(0, 0, 0, 0);
                    uint2 ab = make_uint2(0, 0);
                    if (MU8) ab = *reinterpret_cast<const uint2*>(mask8 + q);
                    else {
                        a0 = *reinterpret_cast<const int4*>(mask32 + q);
                        a1 = *reinterpret_cast<const int4*>(mask32 + q + 4);
                    }
                    const uint4 d = *reinterpret_cast<const uint4*>(dy + q);
                    uint4 tt = make_uint4(0, 0, 0, 0);
                    if (top) tt = *reinterpret_cast<const uint4*>(top + q);
                    window(py, px, a0, a1, ab, d, tt);
                }
        }
#pragma unroll
        for (int i = 0; i < SH; i++)
#pragma unroll
            for (int j = 0; j < SW; j++)
                if (h0 + i < g.H && w0 + j < g.W)
                    *reinterpret_cast<uint4*>(dx + (((long long)n * g.H + h0 + i) * g.W + w0 + j) * g.C + c0) =
                        pack8(acc[i][j]);
    }
}

// ---- 3x3 / stride-2 / unpadded windows that all lie inside the image (every CaffeNet pool: 55->27,
// 27->13, 13->6).  The general kernels above spend ~1.4k instructions per thread on runtime window
// geometry and are issue-bound at 2-3x the HBM time; here the geometry is compile-time.
//
// Forward: thread = one window x 8 channels; the same packed strict-'>' scan as maxpool_fwd_nhwc8
// (first element seeds, NaN never wins), the local index i*3+j being the U8 mask byte directly.
__global__ void maxpool_fwd_k3s2_nhwc8(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                       uint8_t* __restrict__ mask, PoolGeom g, int total) {
    const int cv = g.C / 8;
    GRID_STRIDE(t, total) {
        const int c0 = (t % cv) * 8;
        int r = t / cv;
        const int px = r % g.OW; r /= g.OW;
        const int py = r % g.OH;
        const int n = r / g.OH;
        const __nv_bfloat16* base = x + (((long long)n * g.H + 2 * py) * g.W + 2 * px) * g.C + c0;
        const long long rs = (long long)g.W * g.C;
        uint4 raw[3][3];
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) raw[i][j] = __ldg(reinterpret_cast<const uint4*>(base + i * rs + j * g.C));
        uint32_t bw[4] = {raw[0][0].x, raw[0][0].y, raw[0][0].z, raw[0][0].w};
        uint32_t aw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
                if (i == 0 && j == 0) continue;
                const uint32_t vw[4] = {raw[i][j].x, raw[i][j].y, raw[i][j].z, raw[i][j].w};
                const uint32_t pp = (uint32_t)(i * 3 + j) * 0x00010001u;
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vw[e]),
                                                   *reinterpret_cast<const __nv_bfloat162*>(&bw[e]));
                    bw[e] = (vw[e] & m) | (bw[e] & ~m);
                    aw[e] = (pp & m) | (aw[e] & ~m);
                }
            }
        const long long o = (long long)t * 8;
        *reinterpret_cast<uint4*>(y + o) = make_uint4(bw[0], bw[1], bw[2], bw[3]);
        if (mask)   // 16-bit lane indices (< 9) -> bytes
            *reinterpret_cast<uint2*>(mask + o) = make_uint2(__byte_perm(aw[0], aw[1], 0x6420),
                                                             __byte_perm(aw[2], aw[3], 0x6420));
    }
}

// Backward: a thread owns a column strip of 2x2 blocks of input positions (block (bh, bw) = rows
// 2bh, 2bh+1; cols 2bw, 2bw+1) x 8 channels and walks it downwards.  The windows overlapping block
// (bh, bw) are W11 = (bh-1, bw-1), W10 = (bh-1, bw), W01 = (bh, bw-1), W00 = (bh, bw) -- ascending
// (py, px), R8's order -- so the lower pair of one block is the upper pair of the next: each window
// row is fetched once per strip (plus one row per strip start) instead of twice, and the next row's
// pair is prefetched while the current block is summed.  The window-local index of each block
// position is fixed: (0,0) is 8 / 6 / 2 / 0 in the four windows, (0,1) is 7 in W10 and 1 in W00,
// (1,0) is 5 in W01 and 3 in W00, (1,1) is 4 in W00.  A missing window contributes nothing (mask
// 0xFF).  RELU: the window's gradient passes only when its max y > 0 (packed bf16 compare, false
// for NaN) -- the fused ReLU backward.  Adding a masked-out +0 leaves an FP32 sum unchanged, so the
// straight-line sums equal the hit-only sums of maxpool_bwd_kernel bit for bit.
struct PoolWin {
    uint4 d, y;
    uint2 m;
};

// window at element offset q (valid) or the empty window (mask 0xFF: no position selected)
template <bool RELU>
__device__ __forceinline__ void pool_win_load(PoolWin& w, const __nv_bfloat16* __restrict__ dy,
                                              const uint8_t* __restrict__ mask, const __nv_bfloat16* __restrict__ top,
                                              long long q, bool valid) {
    w.d = make_uint4(0u, 0u, 0u, 0u);
    w.y = make_uint4(0u, 0u, 0u, 0u);
    w.m = make_uint2(0xffffffffu, 0xffffffffu);
    if (valid) {
        w.d = __ldg(reinterpret_cast<const uint4*>(dy + q));
        w.m = __ldg(reinterpret_cast<const uint2*>(mask + q));
        if (RELU) w.y = __ldg(reinterpret_cast<const uint4*>(top + q));
    }
}

template <bool RELU>
__device__ __forceinline__ uint32_t pool_gate(uint32_t d, uint32_t y) {
    if (!RELU) return d;
    return d & __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&y), __float2bfloat162_rn(0.f));
}

__device__ __forceinline__ uint32_t bf2_bits(__nv_bfloat162 v) { return *reinterpret_cast<const uint32_t*>(&v); }
__device__ __forceinline__ __nv_bfloat162 bits_bf2(uint32_t v) { return *reinterpret_cast<const __nv_bfloat162*>(&v); }

// One 2x2 block from its four windows W11, W10, W01, W00 (ascending (py, px), R8's order); the
// window-local index of each block position is fixed: (0,0) is 8 / 6 / 2 / 0 in the four windows,
// (0,1) is 7 in W10 and 1 in W00, (1,0) is 5 in W01 and 3 in W00, (1,1) is 4 in W00.
template <bool RELU>
__device__ __forceinline__ void pool_block_k3s2(const PoolWin& w11, const PoolWin& w10, const PoolWin& w01,
                                                const PoolWin& w00, __nv_bfloat16* o, long long rs, int C, bool right,
                                                bool lower) {
    const PoolWin* W[4] = {&w11, &w10, &w01, &w00};
    // sel(k, t, q): bf16 pair q of window k where the mask byte == t, else +0.  The pair's two mask
    // bytes are XORed with t and moved into the high byte of each 16-bit lane (0x0000 iff equal;
    // otherwise a normal number or NaN -- never -0 or subnormal -- as bf16), and a packed bf16
    // == 0 compare turns that into the lane mask.
    auto sel = [&](int k, uint32_t t, int q) -> uint32_t {
        const uint32_t x = ((q < 2) ? W[k]->m.x : W[k]->m.y) ^ (t * 0x01010101u);
        const uint32_t sp = __byte_perm(x, 0u, (q & 1) ? 0x3424 : 0x1404);
        const uint32_t dq = q == 0 ? W[k]->d.x : q == 1 ? W[k]->d.y : q == 2 ? W[k]->d.z : W[k]->d.w;
        const uint32_t yq = q == 0 ? W[k]->y.x : q == 1 ? W[k]->y.y : q == 2 ? W[k]->y.z : W[k]->y.w;
        return pool_gate<RELU>(dq, yq) & __heq2_mask(bits_bf2(sp), __float2bfloat162_rn(0.f));
    };
    const __nv_bfloat162 z2 = __float2bfloat162_rn(0.f);
    uint32_t o00[4], o01[4], o10[4], o11[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        // (0,0): four windows -> FP32 sum in R8's order, one rounding
        const uint32_t s0 = sel(0, 8, q), s1 = sel(1, 6, q), s2 = sel(2, 2, q), s3 = sel(3, 0, q);
        float lo = 0.f, hi = 0.f;
        lo += __uint_as_float(s0 << 16); hi += __uint_as_float(s0 & 0xffff0000u);
        lo += __uint_as_float(s1 << 16); hi += __uint_as_float(s1 & 0xffff0000u);
        lo += __uint_as_float(s2 << 16); hi += __uint_as_float(s2 & 0xffff0000u);
        lo += __uint_as_float(s3 << 16); hi += __uint_as_float(s3 & 0xffff0000u);
        o00[q] = bf2_bits(__floats2bfloat162_rn(lo, hi));
        // (0,1), (1,0): two windows.  RN_bf16(RN_fp32(a + b)) == RN_bf16(a + b) for two bf16 addends
        // (when a + b is inexact in FP32 the smaller is below 2^-9 ulp_bf16 of the larger), so a
        // packed bf16 add gives R8's result; the trailing + (+0) maps (-0) + (-0) to R8's +0.
        o01[q] = bf2_bits(__hadd2(__hadd2(bits_bf2(sel(1, 7, q)), bits_bf2(sel(3, 1, q))), z2));
        o10[q] = bf2_bits(__hadd2(__hadd2(bits_bf2(sel(2, 5, q)), bits_bf2(sel(3, 3, q))), z2));
        // (1,1): one window; + (+0) as R8's 0 + v
        o11[q] = bf2_bits(__hadd2(bits_bf2(sel(3, 4, q)), z2));
    }
    *reinterpret_cast<uint4*>(o) = make_uint4(o00[0], o00[1], o00[2], o00[3]);
    if (right) *reinterpret_cast<uint4*>(o + C) = make_uint4(o01[0], o01[1], o01[2], o01[3]);
    if (lower) {
        *reinterpret_cast<uint4*>(o + rs) = make_uint4(o10[0], o10[1], o10[2], o10[3]);
        if (right) *reinterpret_cast<uint4*>(o + rs + C) = make_uint4(o11[0], o11[1], o11[2], o11[3]);
    }
}

// Backward: a thread owns a column strip of 2x2 blocks of input positions (block (bh, bw) = rows
// 2bh, 2bh+1; cols 2bw, 2bw+1) x 8 channels and walks it downwards.  Block (bh, bw) reads windows
// (bh-1, bw-1), (bh-1, bw), (bh, bw-1), (bh, bw), so the lower pair of one block is the upper pair
// of the next: each window row is fetched once per strip (plus one row per strip start) instead
// of twice, and the next pair is in flight while the current block is summed (three pair slots,
// rotated by a 3x unrolled loop, so the rotation costs no register moves).  A missing window
// contributes nothing.  RELU: a window's gradient passes only when its max y > 0 (packed bf16
// compare, false for NaN) -- the fused ReLU backward.  Adding a masked-out +0 leaves the sums
// unchanged, so the straight-line sums equal maxpool_bwd_kernel's hit-only sums bit for bit.
template <bool RELU>
__global__ void maxpool_bwd_k3s2_nhwc8(const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ mask,
                                       const __nv_bfloat16* __restrict__ top, __nv_bfloat16* __restrict__ dx,
                                       PoolGeom g, int HB, int WB, int rows, int nstrip, int total) {
    const unsigned cv = (unsigned)g.C / 8u;
    const long long wrs = (long long)g.OW * g.C;   // window row stride
    const long long rs = (long long)g.W * g.C;     // input row stride
    GRID_STRIDE(t, total) {
        const int c0 = (int)((unsigned)t % cv) * 8;
        unsigned r = (unsigned)t / cv;
        const int bw = (int)(r % (unsigned)WB); r /= (unsigned)WB;
        const int st = (int)(r % (unsigned)nstrip);
        const int n = (int)(r / (unsigned)nstrip);
        const int bh0 = st * rows, bh1 = min(bh0 + rows, HB);
        const bool lv = bw >= 1, rv = bw < g.OW;
        // element offset of window (py, bw) -- (py, bw-1) is one C before
        const long long q0 = ((long long)n * g.OH * g.OW + bw) * g.C + c0;
        auto load_pair = [&](PoolWin& a, PoolWin& b, int py) {
            const bool yv = py >= 0 && py < g.OH;
            const long long q = q0 + (long long)py * wrs;
            pool_win_load<RELU>(a, dy, mask, top, q - g.C, yv && lv);
            pool_win_load<RELU>(b, dy, mask, top, q, yv && rv);
        };
        PoolWin A0, A1, B0, B1, C0, C1;
        load_pair(A0, A1, bh0 - 1);
        load_pair(B0, B1, bh0);
        __nv_bfloat16* o = dx + (((long long)n * g.H + 2 * bh0) * g.W + 2 * bw) * g.C + c0;
        const bool right = 2 * bw + 1 < g.W;
        // step: block bh from upper pair (u0, u1) and lower pair (l0, l1), prefetching row bh+1 into (p0, p1)
        auto step = [&](const PoolWin& u0, const PoolWin& u1, const PoolWin& l0, const PoolWin& l1, PoolWin& p0,
                        PoolWin& p1, int bh) {
            load_pair(p0, p1, bh + 1 < bh1 ? bh + 1 : -1);
            pool_block_k3s2<RELU>(u0, u1, l0, l1, o, rs, g.C, right, 2 * bh + 1 < g.H);
            o += 2 * rs;
        };
        for (int bh = bh0; bh < bh1; bh += 3) {
            step(A0, A1, B0, B1, C0, C1, bh);
            if (bh + 1 >= bh1) break;
            step(B0, B1, C0, C1, A0, A1, bh + 1);
            if (bh + 2 >= bh1) break;
            step(C0, C1, A0, A1, B0, B1, bh + 2);
        }
    }
}

// FP32 channels-last 3x3/s2 max-pool backward (the TF32 path's activations): thread = one 2x2 block of
// input positions x 4 channels; its four windows W11, W10, W01, W00 (ascending (py, px)) are read
// once and each position sums the windows that selected it in that order from +0 in FP32 -- R8's
// gather, bit-exact.  RELU: a window passes its gradient only when its max (top) is > 0.
template <bool RELU>
__global__ void maxpool_bwd_k3s2_f32(const float* __restrict__ dy, const uint8_t* __restrict__ mask,
                                     const float* __restrict__ top, float* __restrict__ dx, PoolGeom g, int HB, int WB,
                                     int total) {
    const int cv = g.C / 4;
    GRID_STRIDE(t, total) {
        const int c0 = (t % cv) * 4;
        int r = t / cv;
        const int bw = r % WB; r /= WB;
        const int bh = r % HB;
        const int n = r / HB;
        float4 d[4];
        uint32_t m[4];
#pragma unroll
        for (int w = 0; w < 4; w++) {
            const int py = bh - 1 + (w >> 1), px = bw - 1 + (w & 1);
            d[w] = make_float4(0.f, 0.f, 0.f, 0.f);
            m[w] = 0xffffffffu;
            if (py >= 0 && py < g.OH && px >= 0 && px < g.OW) {
                const long long q = (((long long)n * g.OH + py) * g.OW + px) * g.C + c0;
                d[w] = __ldg(reinterpret_cast<const float4*>(dy + q));
                m[w] = __ldg(reinterpret_cast<const uint32_t*>(mask + q));
                if (RELU) {
                    const float4 y = __ldg(reinterpret_cast<const float4*>(top + q));
                    if (!(y.x > 0.f)) d[w].x = 0.f;
                    if (!(y.y > 0.f)) d[w].y = 0.f;
                    if (!(y.z > 0.f)) d[w].z = 0.f;
                    if (!(y.w > 0.f)) d[w].w = 0.f;
                }
            }
        }
        // window-local index of each block position in W11, W10, W01, W00 (-1: not in the window)
        const int loc[4][4] = {{8, 6, 2, 0}, {-1, 7, -1, 1}, {-1, -1, 5, 3}, {-1, -1, -1, 4}};
#pragma unroll
        for (int pos = 0; pos < 4; pos++) {
            const int h = 2 * bh + (pos >> 1), w_ = 2 * bw + (pos & 1);
            if (h >= g.H || w_ >= g.W) continue;
            float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int w = 0; w < 4; w++) {
                const int l = loc[pos][w];
                if (l < 0) continue;
                const float dv[4] = {d[w].x, d[w].y, d[w].z, d[w].w};
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if ((int)((m[w] >> (8 * e)) & 0xffu) == l) a[e] += dv[e];
            }
            *reinterpret_cast<float4*>(dx + (((long long)n * g.H + h) * g.W + w_) * g.C + c0) =
                make_float4(a[0], a[1], a[2], a[3]);
        }
    }
}

int g_pool_strip_rows = 0;

static inline bool k3s2_full(const PoolGeom& g) {
    return g.kh == 3 && g.kw == 3 && g.sh == 2 && g.sw == 2 && g.ph == 0 && g.pw == 0 && 2 * (g.OH - 1) + 3 <= g.H &&
           2 * (g.OW - 1) + 3 <= g.W && g.H <= 2 * g.OH + 1 && g.W <= 2 * g.OW + 1;
}

static inline bool nhwc8_ok(const void* a, const void* b, int C) {
    return (C % 8) == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
}

cudaError_t maxpool_fwd(const void* x, L4 lx, void* y, int ynhwc, void* mask, int mask_u8, int bf16,
                        const PoolGeom& g, cudaStream_t s) {
    const int total = g.N * g.C * g.OH * g.OW;
    const bool xnhwc = lx.sc == 1 && g.C > 1;
    if (bf16 && xnhwc && ynhwc && nhwc8_ok(x, y, g.C) && ((reinterpret_cast<uintptr_t>(mask) & 15) == 0)) {
        auto X = (const __nv_bfloat16*)x;
        auto Y = (__nv_bfloat16*)y;
        const unsigned nb = nblk(total / 8, 256);
        if (k3s2_full(g) && (mask_u8 || !mask))
            maxpool_fwd_k3s2_nhwc8<<<nb, 256, 0, s>>>(X, Y, (uint8_t*)mask, g, total / 8);
        else if (g.kh == 3 && g.kw == 3) maxpool_fwd_nhwc8<3, 3><<<nb, 256, 0, s>>>(X, Y, mask, mask_u8, g, total / 8);
        else if (g.kh == 2 && g.kw == 2) maxpool_fwd_nhwc8<2, 2><<<nb, 256, 0, s>>>(X, Y, mask, mask_u8, g, total / 8);
        else maxpool_fwd_nhwc8<0, 0><<<nb, 256, 0, s>>>(X, Y, mask, mask_u8, g, total / 8);
    } else {
        maxpool_fwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, lx, y, ynhwc, mask, mask_u8, bf16, g, total);
    }
    note_launch();
    return cudaGetLastError();
}

// Backward: gather per input element (in the bottom_diff's memory order) over the windows that may
// contain it, ascending (py, px) -- R8, bit-exact.  ly = layout strides of top_diff and mask.
__global__ void maxpool_bwd_kernel(const void* __restrict__ dy, const void* __restrict__ mask, int mask_u8,
                                   const void* __restrict__ top, L4 ly, void* __restrict__ dx, int xnhwc, int bf16,
                                   PoolGeom g, int total) {
    GRID_STRIDE(t, total) {
        int n, c, h, w;
        decode(t, g.C, g.H, g.W, xnhwc, n, c, h, w);
        const int py0 = max(0, (h + g.ph - g.kh + g.sh) / g.sh), py1 = min(g.OH - 1, (h + g.ph) / g.sh);
        const int px0 = max(0, (w + g.pw - g.kw + g.sw) / g.sw), px1 = min(g.OW - 1, (w + g.pw) / g.sw);
        const int me = h * g.W + w;
        const int base = n * ly.sn + c * ly.sc;
        float acc = 0.f;
        for (int py = py0; py <= py1; py++)
            for (int px = px0; px <= px1; px++) {
                const int q = base + py * ly.sh + px * ly.sw;
                const bool hit = mask_u8 ? reinterpret_cast<const uint8_t*>(mask)[q] ==
                                               (h - (py * g.sh - g.ph)) * g.kw + (w - (px * g.sw - g.pw))
                                         : reinterpret_cast<const int32_t*>(mask)[q] == me;
                if (hit && (!top || ldv(top, q, bf16) > 0.f)) acc += ldv(dy, q, bf16);
            }
        stv(dx, t, bf16, acc);
    }
}

cudaError_t maxpool_bwd(const void* dy, const void* mask, int mask_u8, const void* top, L4 ly, void* dx, int xnhwc,
                        int bf16, const PoolGeom& g, cudaStream_t s) {
    const int total = g.N * g.C * g.H * g.W;
    const bool ynhwc = ly.sc == 1 && g.C > 1;
    if (bf16 && xnhwc && ynhwc && nhwc8_ok(dy, dx, g.C) && ((reinterpret_cast<uintptr_t>(mask) & 15) == 0) &&
        ((reinterpret_cast<uintptr_t>(top) & 15) == 0)) {
        auto DY = (const __nv_bfloat16*)dy;
        auto T = (const __nv_bfloat16*)top;
        auto DX = (__nv_bfloat16*)dx;
        const int HB = (g.H + 1) / 2, WB = (g.W + 1) / 2, tb = g.N * HB * WB * (g.C / 8);
        if (mask_u8 && k3s2_full(g)) {
            const uint8_t* M = (const uint8_t*)mask;
            // strips of 4 block rows (measured best of 1..28 on pool1/pool2): window rows fetched 5/4
            // times instead of twice, with enough strips in flight to cover HBM latency
            const int rows = g_pool_strip_rows > 0 ? g_pool_strip_rows : (HB >= 7 ? 4 : HB);
            const int nstrip = (HB + rows - 1) / rows, ts = g.N * nstrip * WB * (g.C / 8);
            if (top) maxpool_bwd_k3s2_nhwc8<true><<<nblk(ts, 256), 256, 0, s>>>(DY, M, T, DX, g, HB, WB, rows, nstrip, ts);
            else maxpool_bwd_k3s2_nhwc8<false><<<nblk(ts, 256), 256, 0, s>>>(DY, M, T, DX, g, HB, WB, rows, nstrip, ts);
        } else if (g.sh == 2 && g.sw == 2 && g.kh <= 3 && g.kw <= 3) {
            // a 2x2 block of positions overlaps at most 2x2 windows of size <= 3
            if (mask_u8) maxpool_bwd_nhwc8<2, 2, 2, 2, true><<<nblk(tb, 256), 256, 0, s>>>(DY, mask, T, DX, g, HB, WB, tb);
            else maxpool_bwd_nhwc8<2, 2, 2, 2, false><<<nblk(tb, 256), 256, 0, s>>>(DY, mask, T, DX, g, HB, WB, tb);
        } else if (g.sh == 2 && g.sw == 2) {
            if (mask_u8) maxpool_bwd_nhwc8<2, 2, 0, 0, true><<<nblk(tb, 256), 256, 0, s>>>(DY, mask, T, DX, g, HB, WB, tb);
            else maxpool_bwd_nhwc8<2, 2, 0, 0, false><<<nblk(tb, 256), 256, 0, s>>>(DY, mask, T, DX, g, HB, WB, tb);
        } else {
            if (mask_u8)
                maxpool_bwd_nhwc8<1, 1, 0, 0, true><<<nblk(total / 8, 256), 256, 0, s>>>(DY, mask, T, DX, g, g.H, g.W,
                                                                                     total / 8);
            else
                maxpool_bwd_nhwc8<1, 1, 0, 0, false><<<nblk(total / 8, 256), 256, 0, s>>>(DY, mask, T, DX, g, g.H, g.W,
                                                                                      total / 8);
        }
    } else if (!bf16 && xnhwc && ynhwc && mask_u8 && k3s2_full(g) && g.C % 4 == 0 &&
               ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx) | reinterpret_cast<uintptr_t>(top) |
                 reinterpret_cast<uintptr_t>(mask)) & 15) == 0 && ((reinterpret_cast<uintptr_t>(mask) & 3) == 0)) {
        const int HB = (g.H + 1) / 2, WB = (g.W + 1) / 2, tb = g.N * HB * WB * (g.C / 4);
        if (top)
            maxpool_bwd_k3s2_f32<true><<<nblk(tb, 256), 256, 0, s>>>((const float*)dy, (const uint8_t*)mask,
                                                                      (const float*)top, (float*)dx, g, HB, WB, tb);
        else
            maxpool_bwd_k3s2_f32<false><<<nblk(tb, 256), 256, 0, s>>>((const float*)dy, (const uint8_t*)mask, nullptr,
                                                                       (float*)dx, g, HB, WB, tb);
    } else {
        maxpool_bwd_kernel<<<nblk(total, 256), 256, 0, s>>>(dy, mask, mask_u8, top, ly, dx, xnhwc, bf16, g, total);
    }
    note_launch();
    return cudaGetLastError();
}

__device__ __forceinline__ void ave_window(int py, int px, const PoolGeom& g, int& hs, int& he, int& ws, int& we,
                                           int& size) {
    hs = py * g.sh - g.ph;
    ws = px * g.sw - g.pw;
    he = min(hs + g.kh, g.H + g.ph);
    we = min(ws + g.kw, g.W + g.pw);
    size = (he - hs) * (we - ws);
    hs = max(hs, 0);
    ws = max(ws, 0);
    he = min(he, g.H);
    we = min(we, g.W);
}

__global__ void avepool_fwd_kernel(const void* __restrict__ x, L4 lx, void* __restrict__ y, int ynhwc, int bf16,
                                   PoolGeom g, int total) {
    GRID_STRIDE(t, total) {
        int n, c, py, px;
        decode(t, g.C, g.OH, g.OW, ynhwc, n, c, py, px);
        int hs, he, ws, we, size;
        ave_window(py, px, g, hs, he, ws, we, size);
        const int base = n * lx.sn + c * lx.sc;
        float acc = 0.f;
        for (int h = hs; h < he; h++)
            for (int w = ws; w < we; w++) acc += ldv(x, base + h * lx.sh + w * lx.sw, bf16);
        stv(y, t, bf16, acc / size);
    }
}

cudaError_t avepool_fwd(const void* x, L4 lx, void* y, int ynhwc, int bf16, const PoolGeom& g, cudaStream_t s) {
    const int total = g.N * g.C * g.OH * g.OW;
    avepool_fwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, lx, y, ynhwc, bf16, g, total);
    note_launch();
    return cudaGetLastError();
}

__global__ void avepool_bwd_kernel(const void* __restrict__ dy, L4 ly, void* __restrict__ dx, int xnhwc, int bf16,
                                   PoolGeom g, int total) {
    GRID_STRIDE(t, total) {
        int n, c, h, w;
        decode(t, g.C, g.H, g.W, xnhwc, n, c, h, w);
        const int py0 = max(0, (h + g.ph - g.kh + g.sh) / g.sh), py1 = min(g.OH - 1, (h + g.ph) / g.sh);
        const int px0 = max(0, (w + g.pw - g.kw + g.sw) / g.sw), px1 = min(g.OW - 1, (w + g.pw) / g.sw);
        const int base = n * ly.sn + c * ly.sc;
        float acc = 0.f;
        for (int py = py0; py <= py1; py++)
            for (int px = px0; px <= px1; px++) {
                int hs, he, ws, we, size;
                ave_window(py, px, g, hs, he, ws, we, size);
                if (h >= hs && h < he && w >= ws && w < we) acc += ldv(dy, base + py * ly.sh + px * ly.sw, bf16) / size;
            }
        stv(dx, t, bf16, acc);
    }
}

cudaError_t avepool_bwd(const void* dy, L4 ly, void* dx, int xnhwc, int bf16, const PoolGeom& g, cudaStream_t s) {
    const int total = g.N * g.C * g.H * g.W;
    avepool_bwd_kernel<<<nblk(total, 256), 256, 0, s>>>(dy, ly, dx, xnhwc, bf16, g, total);
    note_launch();
    return cudaGetLastError();
}

// ================================================================ LRN across channels
// All LRN blobs share one layout (checked by the ABI); sc = channel stride.
__device__ __forceinline__ float lrn_scale(const void* x, int bf16, int base, int sc, int c, int C, int r,
                                           float alpha_n, float k) {
    float s = 0.f;
    const int lo = max(0, c - r), hi = min(C - 1, c + r);
    for (int cc = lo; cc <= hi; cc++) {
        const float v = ldv(x, base + cc * sc, bf16);
        s = fmaf(v, v, s);
    }
    return k + alpha_n * s;
}

__global__ void lrn_fwd_kernel(const void* __restrict__ x, void* __restrict__ y, float* __restrict__ scale, int bf16,
                               int nhwc, int C, int H, int W, int sc, int size, float alpha, float beta, float k,
                               int total) {
    const int r = (size - 1) / 2;
    const float an = alpha / size;
    GRID_STRIDE(t, total) {
        int n, c, h, w;
        decode(t, C, H, W, nhwc, n, c, h, w);
        const int base = t - c * sc;
        const float S = lrn_scale(x, bf16, base, sc, c, C, r, an, k);
        stv(y, t, bf16, ldv(x, t, bf16) * exp2f(-beta * log2f(S)));
        if (scale) scale[t] = S;
    }
}

// 8 consecutive channel values as floats / back (BF16: one 16-byte vector; FP32: two)
__device__ __forceinline__ void ld8v(const __nv_bfloat16* p, float (&f)[8]) { unpack8(*reinterpret_cast<const uint4*>(p), f); }
__device__ __forceinline__ void ld8v(const float* p, float (&f)[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
__device__ __forceinline__ void st8v(__nv_bfloat16* p, const float (&f)[8]) { *reinterpret_cast<uint4*>(p) = pack8(f); }
__device__ __forceinline__ void st8v(float* p, const float (&f)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}
// FP32 channels-last LRN (the TF32 path's activations): the same neighbour-vector form
__device__ __forceinline__ void load24(const float* p, int c0, int C, float (&v)[24]) {
    float a[8], b[8], c[8];
    ld8v(p + c0, b);
    if (c0 >= 8) ld8v(p + c0 - 8, a);
    else {
#pragma unroll
        for (int e = 0; e < 8; e++) a[e] = 0.f;
    }
    if (c0 + 8 < C) ld8v(p + c0 + 8, c);
    else {
#pragma unroll
        for (int e = 0; e < 8; e++) c[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < 8; e++) { v[e] = a[e]; v[8 + e] = b[e]; v[16 + e] = c[e]; }
}

// channels-last BF16 LRN: a thread owns 8 channels of one pixel and keeps the neighbouring 8-channel
// vectors (c0-8 .. c0+15) in registers; channels outside [0, C) contribute 0 (clipped window).
__device__ __forceinline__ void load24(const __nv_bfloat16* p, int c0, int C, float (&v)[24]) {
    float a[8], b[8], c[8];
    unpack8(*reinterpret_cast<const uint4*>(p + c0), b);
    if (c0 >= 8) unpack8(*reinterpret_cast<const uint4*>(p + c0 - 8), a);
    else {
#pragma unroll
        for (int e = 0; e < 8; e++) a[e] = 0.f;
    }
    if (c0 + 8 < C) unpack8(*reinterpret_cast<const uint4*>(p + c0 + 8), c);
    else {
#pragma unroll
        for (int e = 0; e < 8; e++) c[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < 8; e++) { v[e] = a[e]; v[8 + e] = b[e]; v[16 + e] = c[e]; }
}

// MUFU forms without the subnormal range handling of __powf / __fdividef: S >= k > 0 here (k = 1
// in CaffeNet), and the results are rounded to BF16, far above the ~2^-22 error of the approximations.
__device__ __forceinline__ float lg2_ftz(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_ftz(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// the 8 outputs of channels c0..c0+7 from the 24 channels c0-8..c0+15 (zero outside [0, C))
template <int R>
__device__ __forceinline__ void lrn_fwd8(const float (&xv)[24], float an, float beta, float k, float (&out)[8],
                                         float (&S)[8]) {
#pragma unroll
    for (int e = 0; e < 8; e++) {
        float s2 = 0.f;
#pragma unroll
        for (int j = -R; j <= R; j++) s2 = fmaf(xv[8 + e + j], xv[8 + e + j], s2);
        S[e] = k + an * s2;
        out[e] = xv[8 + e] * ex2_ftz(-beta * lg2_ftz(S[e]));
    }
}

template <int R, typename T>
__global__ void lrn_fwd_nhwc8(const T* __restrict__ x, T* __restrict__ y,
                              float* __restrict__ scale, int C, int size, float alpha, float beta, float k, int total) {
    const int cv = C / 8;
    const float an = alpha / size;
    GRID_STRIDE(t, total) {
        const int c0 = (t % cv) * 8;
        const long long base = (long long)(t / cv) * C;
        float xv[24];
        load24(x + base, c0, C, xv);
        float out[8], S[8];
        lrn_fwd8<R>(xv, an, beta, k, out, S);
        st8v(y + base + c0, out);
        if (scale) {
            float4* sp = reinterpret_cast<float4*>(scale + base + c0);
            sp[0] = make_float4(S[0], S[1], S[2], S[3]);
            sp[1] = make_float4(S[4], S[5], S[6], S[7]);
        }
    }
}

// Backward: the window sums over the 8 + 2R channel positions slide (one add and one subtract per
// step); each position takes Q = S^(-beta-1) = 2^((-beta-1) lg2 S) and S^-beta = Q * S: two MUFU
// operations (lg2, ex2) instead of three (no reciprocal; the kernel is issue-bound).  The
// cross-channel term uses y/S = x * Q recomputed in FP32 from the bottom (the stored top is
// BF16-rounded: reading it made the result lose up to 2^-9 of that term where it cancels the direct
// term, and cost a third of the kernel's reads); `y` is not read.  The 8 outputs' window sums of
// dy*y/S slide (one add and one subtract per step); FP32 throughout, BF16 or FP32 output.
template <int R>
__device__ __forceinline__ void lrn_bwd8(const float (&xv)[24], const float (&gv)[24], float an, float beta, float k,
                                         float cb, float (&out)[8]) {
    float P[24], tv[24];
    const float nb1 = -beta - 1.f;
    float s2 = 0.f;
#pragma unroll
    for (int j = 8 - 2 * R; j <= 8; j++) s2 = fmaf(xv[j], xv[j], s2);   // window of channel 8 - R
#pragma unroll
    for (int i = 8 - R; i < 16 + R; i++) {
        if (i > 8 - R) {
            s2 = fmaf(xv[i + R], xv[i + R], s2);
            s2 = fmaf(-xv[i - R - 1], xv[i - R - 1], s2);
        }
        const float S = k + an * s2;
        const float Q = ex2_ftz(nb1 * lg2_ftz(S));           // S^(-beta-1)
        P[i] = Q * S;                                          // S^-beta
        tv[i] = gv[i] * (xv[i] * Q);                           // dy * y / S
    }
    float acc = 0.f;
#pragma unroll
    for (int j = 8 - R; j <= 8 + R; j++) acc += tv[j];
#pragma unroll
    for (int e = 0; e < 8; e++) {
        if (e > 0) acc = acc + tv[8 + e + R] - tv[8 + e - R - 1];
        out[e] = gv[8 + e] * P[8 + e] - cb * xv[8 + e] * acc;
    }
}

template <int R, typename T>
__global__ void lrn_bwd_nhwc8(const T* __restrict__ x, const T* __restrict__ dy,
                              T* __restrict__ dx, int C, int size, float alpha, float beta, float k,
                              int total) {
    const int cv = C / 8;
    const float an = alpha / size;
    const float cb = 2.f * an * beta;
    GRID_STRIDE(t, total) {
        const int c0 = (t % cv) * 8;
        const long long base = (long long)(t / cv) * C;
        float xv[24], gv[24];
        load24(x + base, c0, C, xv);
        load24(dy + base, c0, C, gv);
        float out[8];
        lrn_bwd8<R>(xv, gv, an, beta, k, cb, out);
        st8v(dx + base + c0, out);
    }
}

template <typename T>
static void lrn_fwd_launch(const void* x, void* y, float* scale, int C, int size, float alpha, float beta, float k,
                           int tv, unsigned nb, cudaStream_t s) {
    auto X = (const T*)x;
    auto Y = (T*)y;
    switch ((size - 1) / 2) {
        case 0: lrn_fwd_nhwc8<0, T><<<nb, 256, 0, s>>>(X, Y, scale, C, size, alpha, beta, k, tv); break;
        case 1: lrn_fwd_nhwc8<1, T><<<nb, 256, 0, s>>>(X, Y, scale, C, size, alpha, beta, k, tv); break;
        case 2: lrn_fwd_nhwc8<2, T><<<nb, 256, 0, s>>>(X, Y, scale, C, size, alpha, beta, k, tv); break;
        case 3: lrn_fwd_nhwc8<3, T><<<nb, 256, 0, s>>>(X, Y, scale, C, size, alpha, beta, k, tv); break;
        default: lrn_fwd_nhwc8<4, T><<<nb, 256, 0, s>>>(X, Y, scale, C, size, alpha, beta, k, tv); break;
    }
}

template <typename T>
static void lrn_bwd_launch(const void* x, const void* dy, void* dx, int C, int size, float alpha, float beta, float k,
                           int tv, unsigned nb, cudaStream_t s) {
    auto X = (const T*)x;
    auto G = (const T*)dy;
    auto D = (T*)dx;
    switch ((size - 1) / 2) {
        case 0: lrn_bwd_nhwc8<0, T><<<nb, 256, 0, s>>>(X, G, D, C, size, alpha, beta, k, tv); break;
        case 1: lrn_bwd_nhwc8<1, T><<<nb, 256, 0, s>>>(X, G, D, C, size, alpha, beta, k, tv); break;
        case 2: lrn_bwd_nhwc8<2, T><<<nb, 256, 0, s>>>(X, G, D, C, size, alpha, beta, k, tv); break;
        case 3: lrn_bwd_nhwc8<3, T><<<nb, 256, 0, s>>>(X, G, D, C, size, alpha, beta, k, tv); break;
        default: lrn_bwd_nhwc8<4, T><<<nb, 256, 0, s>>>(X, G, D, C, size, alpha, beta, k, tv); break;
    }
}

cudaError_t lrn_fwd(const void* x, void* y, float* scale, int bf16, int nhwc, int N, int C, int H, int W, int size,
                    float alpha, float beta, float k, cudaStream_t s) {
    const int total = N * C * H * W;
    const int sc = nhwc ? 1 : H * W;
    if (nhwc && nhwc8_ok(x, y, C) && ((reinterpret_cast<uintptr_t>(scale) & 15) == 0) && size <= 9) {
        const int tv = total / 8;
        const unsigned nb = nblk(tv, 256);
        if (bf16) lrn_fwd_launch<__nv_bfloat16>(x, y, scale, C, size, alpha, beta, k, tv, nb, s);
        else lrn_fwd_launch<float>(x, y, scale, C, size, alpha, beta, k, tv, nb, s);
        note_launch();
        return cudaGetLastError();
    }
    lrn_fwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, y, scale, bf16, nhwc, C, H, W, sc, size, alpha, beta, k, total);
    note_launch();
    return cudaGetLastError();
}

__global__ void lrn_bwd_kernel(const void* __restrict__ x, const void* __restrict__ y, const void* __restrict__ dy,
                               const float* __restrict__ scale, void* __restrict__ dx, int bf16, int nhwc, int C, int H,
                               int W, int sc, int size, float alpha, float beta, float k, int total) {
    const int r = (size - 1) / 2;
    const float an = alpha / size;
    GRID_STRIDE(t, total) {
        int n, c, h, w;
        decode(t, C, H, W, nhwc, n, c, h, w);
        const int base = t - c * sc;
        // window sums of x^2 for the 2r+1 neighbours from one pass over 4r+1 channels
        const float Sc = scale ? scale[t] : lrn_scale(x, bf16, base, sc, c, C, r, an, k);
        float acc = 0.f;
        const int lo = max(0, c - r), hi = min(C - 1, c + r);
        for (int cc = lo; cc <= hi; cc++) {
            const int q = base + cc * sc;
            const float S = scale ? scale[q] : lrn_scale(x, bf16, base, sc, cc, C, r, an, k);
            // y/S from the bottom in FP32 (the stored top may be BF16-rounded)
            acc += ldv(dy, q, bf16) * (ldv(x, q, bf16) * exp2f(-beta * log2f(S))) / S;
        }
        const float v = ldv(dy, t, bf16) * exp2f(-beta * log2f(Sc)) - 2.f * an * beta * ldv(x, t, bf16) * acc;
        stv(dx, t, bf16, v);
    }
}

// BF16 channels-last LRN backward with 16 channels per lane (C % 16 == 0, C/16 <= 32): a lane loads
// only its own 16 channels of x and dy (the 8-channel kernel loads 24 of each, neighbours included)
// and takes the neighbouring 8-channel vectors from the adjacent lanes of the same pixel by shuffle;
// each 8-channel half then goes through lrn_bwd8 with exactly the 24 channels the 8-channel kernel
// would have loaded (zero outside [0, C)) -- the same bits.
__device__ __forceinline__ void unpack_words8(const uint32_t* w, float* f) {
#pragma unroll
    for (int e = 0; e < 4; e++) {
        f[2 * e] = __uint_as_float(w[e] << 16);
        f[2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
    }
}
template <int R>
__global__ void __launch_bounds__(256) lrn_bwd_c16(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy,
                                                   __nv_bfloat16* __restrict__ dx, int C, int npix, float an, float beta,
                                                   float k, float cb) {
    const int cv = C / 16, ppw = 32 / cv;
    const int lane = threadIdx.x & 31;
    const int ps = lane / cv, vi = lane - ps * cv;
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int w0 = gw * ppw; w0 < npix; w0 += nw * ppw) {      // warp-uniform loop
        const int pix = w0 + ps;
        const bool act = ps < ppw && pix < npix;
        uint32_t xw[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}, gw8[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        const long long o = (long long)pix * C + vi * 16;
        if (act) {
            const uint4* xp = reinterpret_cast<const uint4*>(x + o);
            const uint4* gp = reinterpret_cast<const uint4*>(dy + o);
            const uint4 x0 = __ldg(xp), x1 = __ldg(xp + 1), g0 = __ldg(gp), g1 = __ldg(gp + 1);
            xw[0] = x0.x; xw[1] = x0.y; xw[2] = x0.z; xw[3] = x0.w; xw[4] = x1.x; xw[5] = x1.y; xw[6] = x1.z; xw[7] = x1.w;
            gw8[0] = g0.x; gw8[1] = g0.y; gw8[2] = g0.z; gw8[3] = g0.w; gw8[4] = g1.x; gw8[5] = g1.y; gw8[6] = g1.z; gw8[7] = g1.w;
        }
        uint32_t xl[4], xr[4], gl[4], gr[4];   // the left lane's upper 8 channels, the right lane's lower 8
#pragma unroll
        for (int e = 0; e < 4; e++) {
            xl[e] = __shfl_up_sync(0xffffffffu, xw[4 + e], 1);
            gl[e] = __shfl_up_sync(0xffffffffu, gw8[4 + e], 1);
            xr[e] = __shfl_down_sync(0xffffffffu, xw[e], 1);
            gr[e] = __shfl_down_sync(0xffffffffu, gw8[e], 1);
        }
        if (vi == 0) { xl[0] = xl[1] = xl[2] = xl[3] = 0u; gl[0] = gl[1] = gl[2] = gl[3] = 0u; }
        if (vi == cv - 1) { xr[0] = xr[1] = xr[2] = xr[3] = 0u; gr[0] = gr[1] = gr[2] = gr[3] = 0u; }
        if (act) {
            float xv[24], gv[24], out[8];
            // half 0: channels c0-8 .. c0+15
            unpack_words8(xl, xv); unpack_words8(xw, xv + 8); unpack_words8(xw + 4, xv + 16);
            unpack_words8(gl, gv); unpack_words8(gw8, gv + 8); unpack_words8(gw8 + 4, gv + 16);
            lrn_bwd8<R>(xv, gv, an, beta, k, cb, out);
            uint4* d = reinterpret_cast<uint4*>(dx + o);
            d[0] = pack8(out);
            // half 1: channels c0 .. c0+23
            unpack_words8(xw, xv); unpack_words8(xw + 4, xv + 8); unpack_words8(xr, xv + 16);
            unpack_words8(gw8, gv); unpack_words8(gw8 + 4, gv + 8); unpack_words8(gr, gv + 16);
            lrn_bwd8<R>(xv, gv, an, beta, k, cb, out);
            d[1] = pack8(out);
        }
    }
}
int g_lrn_bwd_c16 = 1;   // CAFFE_TUNE_LRN_BWD_C16

cudaError_t lrn_bwd(const void* x, const void* y, const void* dy, const float* scale, void* dx, int bf16, int nhwc,
                    int N, int C, int H, int W, int size, float alpha, float beta, float k, cudaStream_t s) {
    const int total = N * C * H * W;
    const int sc = nhwc ? 1 : H * W;
    if (g_lrn_bwd_c16 && nhwc && bf16 && C % 16 == 0 && C / 16 <= 32 && size <= 9 && nhwc8_ok(x, y, C) &&
        nhwc8_ok(dy, dx, C)) {
        const int cv = C / 16, ppw = 32 / cv, npix = N * H * W;
        const long long warps = (npix + ppw - 1) / ppw;
        const unsigned grid = (unsigned)std::max(1LL, std::min((warps * 32 + 255) / 256, 148LL * 16));
        const float an = alpha / size, cbv = 2.f * an * beta;
        auto X = (const __nv_bfloat16*)x;
        auto G = (const __nv_bfloat16*)dy;
        auto D = (__nv_bfloat16*)dx;
        switch ((size - 1) / 2) {
            case 0: lrn_bwd_c16<0><<<grid, 256, 0, s>>>(X, G, D, C, npix, an, beta, k, cbv); break;
            case 1: lrn_bwd_c16<1><<<grid, 256, 0, s>>>(X, G, D, C, npix, an, beta, k, cbv); break;
            case 2: lrn_bwd_c16<2><<<grid, 256, 0, s>>>(X, G, D, C, npix, an, beta, k, cbv); break;
            case 3: lrn_bwd_c16<3><<<grid, 256, 0, s>>>(X, G, D, C, npix, an, beta, k, cbv); break;
            default: lrn_bwd_c16<4><<<grid, 256, 0, s>>>(X, G, D, C, npix, an, beta, k, cbv); break;
        }
        note_launch();
        return cudaGetLastError();
    }
    if (nhwc && nhwc8_ok(x, y, C) && nhwc8_ok(dy, dx, C) && size <= 9) {
        const int tv = total / 8;
        const unsigned nb = nblk(tv, 256);
        if (bf16) lrn_bwd_launch<__nv_bfloat16>(x, dy, dx, C, size, alpha, beta, k, tv, nb, s);
        else lrn_bwd_launch<float>(x, dy, dx, C, size, alpha, beta, k, tv, nb, s);
        note_launch();
        return cudaGetLastError();
    }
    lrn_bwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, y, dy, scale, dx, bf16, nhwc, C, H, W, sc, size, alpha, beta, k,
                                                     total);
    note_launch();
    return cudaGetLastError();
}

// ================================================================ fused max pool + LRN
// CaffeNet's conv -> ReLU -> pool (3x3/s2) -> LRN blocks, BF16 channels-last, U8 window-local mask.
// Both kernels give exactly the bits of the separate calls (the pool's packed strict-'>' scan, the
// LRN arithmetic through the same device functions, R8's FP32 sum order) and drop the
// intermediate blob's trip through HBM.  Layout of the work: the lanes of a warp hold consecutive
// 8-channel vectors of one pooled pixel (C/8 <= 32 lanes per pixel, 32/(C/8) pixels per warp), so
// the cross-channel LRN window is a warp shuffle of the neighbouring lanes' values -- no shared
// memory (the kernels co-reside with the 200 KB tensor-core CTAs of the other streams) and no
// block-wide barrier.
//   forward : pool the warp's pixels (9 loads per lane), store pool output + mask, shuffle the
//             neighbours' pooled values, LRN, store -- the pool output is not re-read;
//   backward: a pixel slot walks a strip of `rows` 2x2-block rows column by column; at each column
//             it computes the LRN backward of the strip's window column (rows+1 pooled pixels: the
//             lanes of the pixel cooperate, neighbours by shuffle), gates it by pool output > 0 (the
//             ReLU below), and runs the max-pool backward of the strip's blocks from that column
//             and the previous one (kept in registers) -- every window's LRN backward is computed
//             once per strip, the LRN bottom diff never reaches memory, the pool output is read once.
__device__ __forceinline__ void shfl_neighbours(const uint32_t (&w)[4], int vi, int cv, float (&xv)[24]) {
    uint32_t l[4], r[4];
#pragma unroll
    for (int e = 0; e < 4; e++) {
        l[e] = __shfl_up_sync(0xffffffffu, w[e], 1);
        r[e] = __shfl_down_sync(0xffffffffu, w[e], 1);
    }
    if (vi == 0) l[0] = l[1] = l[2] = l[3] = 0u;             // channels below 0
    if (vi == cv - 1) r[0] = r[1] = r[2] = r[3] = 0u;        // channels from C up
#pragma unroll
    for (int e = 0; e < 4; e++) {
        xv[2 * e] = __uint_as_float(l[e] << 16);
        xv[2 * e + 1] = __uint_as_float(l[e] & 0xffff0000u);
        xv[8 + 2 * e] = __uint_as_float(w[e] << 16);
        xv[8 + 2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
        xv[16 + 2 * e] = __uint_as_float(r[e] << 16);
        xv[16 + 2 * e + 1] = __uint_as_float(r[e] & 0xffff0000u);
    }
}

template <int R>
__global__ void __launch_bounds__(256)
pool_lrn_fwd_k3s2_nhwc8(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ p, uint8_t* __restrict__ mask,
                        __nv_bfloat16* __restrict__ y, PoolGeom g, int npix, float an, float beta, float k) {
    const int cv = g.C / 8, ppw = 32 / cv;
    const int lane = threadIdx.x & 31;
    const int ps = lane / cv, vi = lane - ps * cv;
    const int c0 = vi * 8;
    const long long rs = (long long)g.W * g.C;
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int w0 = gw * ppw; w0 < npix; w0 += nw * ppw) {      // warp-uniform loop
        const int pix = w0 + ps;
        const bool act = ps < ppw && pix < npix;
        uint32_t bw[4] = {0u, 0u, 0u, 0u}, aw[4] = {0u, 0u, 0u, 0u};
        if (act) {
            int r = pix;
            const int px = r % g.OW; r /= g.OW;
            const int py = r % g.OH;
            const int n = r / g.OH;
            const __nv_bfloat16* base = x + (((long long)n * g.H + 2 * py) * g.W + 2 * px) * g.C + c0;
            uint4 raw[3][3];
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) raw[i][j] = __ldg(reinterpret_cast<const uint4*>(base + i * rs + j * g.C));
            bw[0] = raw[0][0].x; bw[1] = raw[0][0].y; bw[2] = raw[0][0].z; bw[3] = raw[0][0].w;
#pragma unroll
            for (int i = 0; i < 3; i++)
#pragma unroll
                for (int j = 0; j < 3; j++) {
                    if (i == 0 && j == 0) continue;
                    const uint32_t vw[4] = {raw[i][j].x, raw[i][j].y, raw[i][j].z, raw[i][j].w};
                    const uint32_t pp = (uint32_t)(i * 3 + j) * 0x00010001u;
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vw[e]),
                                                       *reinterpret_cast<const __nv_bfloat162*>(&bw[e]));
                        bw[e] = (vw[e] & m) | (bw[e] & ~m);
                        aw[e] = (pp & m) | (aw[e] & ~m);
                    }
                }
            const long long o = (long long)pix * g.C + c0;
            *reinterpret_cast<uint4*>(p + o) = make_uint4(bw[0], bw[1], bw[2], bw[3]);
            *reinterpret_cast<uint2*>(mask + o) =
                make_uint2(__byte_perm(aw[0], aw[1], 0x6420), __byte_perm(aw[2], aw[3], 0x6420));
        }
        float xv[24];
        shfl_neighbours(bw, vi, cv, xv);
        if (act) {
            float out[8], S[8];
            lrn_fwd8<R>(xv, an, beta, k, out, S);
            *reinterpret_cast<uint4*>(y + (long long)pix * g.C + c0) = pack8(out);
        }
    }
}

// the gated LRN bottom diff of pooled pixel (py, px) (own 8 channels) + its mask word; a missing
// window (outside the map) has d = 0 and mask 0xFF (selects no block position)
template <int R, bool RELU>
__device__ __forceinline__ void lrn_window(PoolWin& w, const __nv_bfloat16* __restrict__ p,
                                           const __nv_bfloat16* __restrict__ dn, const uint8_t* __restrict__ mask,
                                           long long q, bool valid, int vi, int cv, float an, float beta, float k,
                                           float cb) {
    uint4 pv = make_uint4(0u, 0u, 0u, 0u), gvv = make_uint4(0u, 0u, 0u, 0u);
    w.m = make_uint2(0xffffffffu, 0xffffffffu);
    w.y = make_uint4(0u, 0u, 0u, 0u);
    if (valid) {
        pv = __ldg(reinterpret_cast<const uint4*>(p + q));
        gvv = __ldg(reinterpret_cast<const uint4*>(dn + q));
        w.m = __ldg(reinterpret_cast<const uint2*>(mask + q));
    }
    const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w}, gw4[4] = {gvv.x, gvv.y, gvv.z, gvv.w};
    float xv[24], gv[24];
    shfl_neighbours(pw, vi, cv, xv);
    shfl_neighbours(gw4, vi, cv, gv);
    float out[8];
    lrn_bwd8<R>(xv, gv, an, beta, k, cb, out);
    uint4 d = valid ? pack8(out) : make_uint4(0u, 0u, 0u, 0u);
    if (RELU) {
        d.x = pool_gate<true>(d.x, pv.x);
        d.y = pool_gate<true>(d.y, pv.y);
        d.z = pool_gate<true>(d.z, pv.z);
        d.w = pool_gate<true>(d.w, pv.w);
    }
    w.d = d;
}

template <int R, bool RELU, int ROWS>
__global__ void __launch_bounds__(256)
lrn_pool_bwd_k3s2_nhwc8(const __nv_bfloat16* __restrict__ p, const __nv_bfloat16* __restrict__ dn,
                        const uint8_t* __restrict__ mask, __nv_bfloat16* __restrict__ dx, PoolGeom g, int HB, int WB,
                        int nstrip, int cseg, int ncseg, int ntask, float an, float beta, float k, float cb) {
    const int cv = g.C / 8, ppw = 32 / cv;
    const int lane = threadIdx.x & 31;
    const int ps = lane / cv, vi = lane - ps * cv;
    const int c0 = vi * 8;
    const long long rs = (long long)g.W * g.C;
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int t0 = gw * ppw; t0 < ntask; t0 += nw * ppw) {     // warp-uniform loop
        const int task = t0 + ps;
        const bool act = ps < ppw && task < ntask;
        // task = ((n * nstrip + strip) * ncseg + column segment); inactive slots mirror slot 0's
        // geometry so the warp's loop trip counts stay uniform (they load and store nothing)
        int tr = act ? task : t0;
        const int seg = tr % ncseg; tr /= ncseg;
        const int st = tr % nstrip;
        const int n = tr / nstrip;
        const int bh0 = st * ROWS;
        const int bw0 = seg * cseg, bw1 = min(bw0 + cseg, WB);
        const long long img = (long long)n * g.OH * g.OW * g.C + c0;
        PoolWin L[ROWS + 1], Rw[ROWS + 1];
        // left window column (bw0 - 1)
#pragma unroll
        for (int a = 0; a <= ROWS; a++) {
            const int py = bh0 - 1 + a, px = bw0 - 1;
            const bool v = act && py >= 0 && py < g.OH && px >= 0 && px < g.OW;
            lrn_window<R, RELU>(L[a], p, dn, mask, img + ((long long)py * g.OW + px) * g.C, v, vi, cv, an, beta, k, cb);
        }
        for (int bw = bw0; bw < bw1; bw++) {
#pragma unroll
            for (int a = 0; a <= ROWS; a++) {
                const int py = bh0 - 1 + a;
                const bool v = act && py >= 0 && py < g.OH && bw < g.OW;
                lrn_window<R, RELU>(Rw[a], p, dn, mask, img + ((long long)py * g.OW + bw) * g.C, v, vi, cv, an, beta, k,
                                    cb);
            }
            if (act) {
                const bool right = 2 * bw + 1 < g.W;
#pragma unroll
                for (int a = 0; a < ROWS; a++) {
                    const int bh = bh0 + a;
                    if (bh < HB) {
                        __nv_bfloat16* o = dx + (((long long)n * g.H + 2 * bh) * g.W + 2 * bw) * g.C + c0;
                        pool_block_k3s2<false>(L[a], Rw[a], L[a + 1], Rw[a + 1], o, rs, g.C, right, 2 * bh + 1 < g.H);
                    }
                }
            }
#pragma unroll
            for (int a = 0; a <= ROWS; a++) L[a] = Rw[a];
        }
    }
}

int g_fused_rb = 0;   // CAFFE_TUNE_FUSED_POOL_ROWS: block rows per strip of the fused backward (0 = automatic)

bool pool_lrn_fusable(const PoolGeom& g, int size) {
    return k3s2_full(g) && g.C % 8 == 0 && g.C / 8 <= 32 && size <= 9 && size % 2 == 1;
}

static unsigned warps_grid(long long warps) {
    long long b = (warps * 32 + 255) / 256;
    const long long cap = 148LL * 16;
    return (unsigned)std::max(1LL, std::min(b, cap));
}

// 16 channels per lane (C % 16 == 0, LRN window radius <= 2): C/16 lanes per pooled pixel (6 for
// CaffeNet's 96-channel norm1: 5 pixels = 30 active lanes per warp, where the 8-channel form idles a
// quarter of them), 18 window loads in flight per lane; the LRN window needs 2 channels from each
// neighbouring lane (one bf16x2 word by shuffle).  Pool scan and LRN arithmetic as in the 8-channel
// kernel (and the separate calls), so the bits are the same.
__device__ __forceinline__ void pool9_scan8(const __nv_bfloat16* base, long long rs, int C, uint32_t (&bw)[4],
                                            uint32_t (&aw)[4]) {
    uint4 raw[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) raw[i][j] = __ldg(reinterpret_cast<const uint4*>(base + i * rs + j * C));
    bw[0] = raw[0][0].x; bw[1] = raw[0][0].y; bw[2] = raw[0][0].z; bw[3] = raw[0][0].w;
    aw[0] = aw[1] = aw[2] = aw[3] = 0u;
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
            if (i == 0 && j == 0) continue;
            const uint32_t vw[4] = {raw[i][j].x, raw[i][j].y, raw[i][j].z, raw[i][j].w};
            const uint32_t pp = (uint32_t)(i * 3 + j) * 0x00010001u;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vw[e]),
                                               *reinterpret_cast<const __nv_bfloat162*>(&bw[e]));
                bw[e] = (vw[e] & m) | (bw[e] & ~m);
                aw[e] = (pp & m) | (aw[e] & ~m);
            }
        }
}

template <int R>
__global__ void __launch_bounds__(256)
pool_lrn_fwd_k3s2_c16(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ p, uint8_t* __restrict__ mask,
                      __nv_bfloat16* __restrict__ y, PoolGeom g, int npix, float an, float beta, float k) {
    static_assert(R <= 2, "two channels from each neighbouring lane");
    const int cv = g.C / 16, ppw = 32 / cv;
    const int lane = threadIdx.x & 31;
    const int ps = lane / cv, vi = lane - ps * cv;
    const int c0 = vi * 16;
    const long long rs = (long long)g.W * g.C;
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int w0 = gw * ppw; w0 < npix; w0 += nw * ppw) {      // warp-uniform loop
        const int pix = w0 + ps;
        const bool act = ps < ppw && pix < npix;
        uint32_t bw[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}, aw[8];
        if (act) {
            int r = pix;
            const int px = r % g.OW; r /= g.OW;
            const int py = r % g.OH;
            const int n = r / g.OH;
            const __nv_bfloat16* base = x + (((long long)n * g.H + 2 * py) * g.W + 2 * px) * g.C + c0;
            uint32_t b0[4], a0[4], b1[4], a1[4];
            pool9_scan8(base, rs, g.C, b0, a0);
            pool9_scan8(base + 8, rs, g.C, b1, a1);
#pragma unroll
            for (int e = 0; e < 4; e++) { bw[e] = b0[e]; bw[4 + e] = b1[e]; aw[e] = a0[e]; aw[4 + e] = a1[e]; }
            const long long o = (long long)pix * g.C + c0;
            uint4* po = reinterpret_cast<uint4*>(p + o);
            po[0] = make_uint4(bw[0], bw[1], bw[2], bw[3]);
            po[1] = make_uint4(bw[4], bw[5], bw[6], bw[7]);
            uint2* mo = reinterpret_cast<uint2*>(mask + o);
            mo[0] = make_uint2(__byte_perm(aw[0], aw[1], 0x6420), __byte_perm(aw[2], aw[3], 0x6420));
            mo[1] = make_uint2(__byte_perm(aw[4], aw[5], 0x6420), __byte_perm(aw[6], aw[7], 0x6420));
        }
        // channels c0-2, c0-1 (left lane's last word) and c0+16, c0+17 (right lane's first word)
        uint32_t lw = __shfl_up_sync(0xffffffffu, bw[7], 1);
        uint32_t rw = __shfl_down_sync(0xffffffffu, bw[0], 1);
        if (vi == 0) lw = 0u;
        if (vi == cv - 1) rw = 0u;
        if (act) {
            float xv[20];   // channels c0-2 .. c0+17
            xv[0] = __uint_as_float(lw << 16);
            xv[1] = __uint_as_float(lw & 0xffff0000u);
#pragma unroll
            for (int e = 0; e < 8; e++) {
                xv[2 + 2 * e] = __uint_as_float(bw[e] << 16);
                xv[3 + 2 * e] = __uint_as_float(bw[e] & 0xffff0000u);
            }
            xv[18] = __uint_as_float(rw << 16);
            xv[19] = __uint_as_float(rw & 0xffff0000u);
            float out[16];
#pragma unroll
            for (int e = 0; e < 16; e++) {   // lrn_fwd8's arithmetic, element by element
                float s2 = 0.f;
#pragma unroll
                for (int j = -R; j <= R; j++) s2 = fmaf(xv[2 + e + j], xv[2 + e + j], s2);
                const float S = k + an * s2;
                out[e] = xv[2 + e] * ex2_ftz(-beta * lg2_ftz(S));
            }
            float o8a[8], o8b[8];
#pragma unroll
            for (int e = 0; e < 8; e++) { o8a[e] = out[e]; o8b[e] = out[8 + e]; }
            uint4* yo = reinterpret_cast<uint4*>(y + (long long)pix * g.C + c0);
            yo[0] = pack8(o8a);
            yo[1] = pack8(o8b);
        }
    }
}
int g_pool_lrn_c16 = 1;   // CAFFE_TUNE_POOL_LRN_C16

cudaError_t pool_lrn_fwd(const void* x, void* p, void* mask, void* y, const PoolGeom& g, int size, float alpha,
                         float beta, float k, cudaStream_t s) {
    if (g_pool_lrn_c16 && g.C % 16 == 0 && g.C / 16 <= 32 && 32 % (g.C / 8) != 0 && size <= 5) {
        const int cv = g.C / 16, ppw = 32 / cv, npix = g.N * g.OH * g.OW;
        const unsigned grid = warps_grid((npix + ppw - 1) / ppw);
        const float an = alpha / size;
        auto X = (const __nv_bfloat16*)x;
        auto P = (__nv_bfloat16*)p;
        auto Y = (__nv_bfloat16*)y;
        auto M = (uint8_t*)mask;
        switch ((size - 1) / 2) {
            case 0: pool_lrn_fwd_k3s2_c16<0><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
            case 1: pool_lrn_fwd_k3s2_c16<1><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
            default: pool_lrn_fwd_k3s2_c16<2><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
        }
        note_launch();
        return cudaGetLastError();
    }
    const int cv = g.C / 8;
    if (cv > 32) return cudaErrorInvalidValue;
    const int ppw = 32 / cv, npix = g.N * g.OH * g.OW;
    const unsigned grid = warps_grid((npix + ppw - 1) / ppw);
    const float an = alpha / size;
    auto X = (const __nv_bfloat16*)x;
    auto P = (__nv_bfloat16*)p;
    auto Y = (__nv_bfloat16*)y;
    auto M = (uint8_t*)mask;
    switch ((size - 1) / 2) {
        case 0: pool_lrn_fwd_k3s2_nhwc8<0><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
        case 1: pool_lrn_fwd_k3s2_nhwc8<1><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
        case 2: pool_lrn_fwd_k3s2_nhwc8<2><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
        case 3: pool_lrn_fwd_k3s2_nhwc8<3><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
        default: pool_lrn_fwd_k3s2_nhwc8<4><<<grid, 256, 0, s>>>(X, P, M, Y, g, npix, an, beta, k); break;
    }
    note_launch();
    return cudaGetLastError();
}

template <int R, int ROWS>
static void lrn_pool_bwd_rows(bool relu, unsigned grid, cudaStream_t s, const __nv_bfloat16* P, const __nv_bfloat16* DN,
                              const uint8_t* M, __nv_bfloat16* DX, const PoolGeom& g, int HB, int WB, int nstrip,
                              int cseg, int ncseg, int ntask, float an, float beta, float k, float cb) {
    if (relu)
        lrn_pool_bwd_k3s2_nhwc8<R, true, ROWS><<<grid, 256, 0, s>>>(P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask,
                                                                     an, beta, k, cb);
    else
        lrn_pool_bwd_k3s2_nhwc8<R, false, ROWS><<<grid, 256, 0, s>>>(P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask,
                                                                      an, beta, k, cb);
}

template <int R>
static void lrn_pool_bwd_r(int rows, bool relu, unsigned grid, cudaStream_t s, const __nv_bfloat16* P,
                           const __nv_bfloat16* DN, const uint8_t* M, __nv_bfloat16* DX, const PoolGeom& g, int HB,
                           int WB, int nstrip, int cseg, int ncseg, int ntask, float an, float beta, float k, float cb) {
    if (rows == 1) lrn_pool_bwd_rows<R, 1>(relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb);
    else if (rows == 2) lrn_pool_bwd_rows<R, 2>(relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb);
    else lrn_pool_bwd_rows<R, 4>(relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb);
}

cudaError_t lrn_pool_bwd(const void* p, const void* dn, const void* mask, void* dx, int relu, const PoolGeom& g,
                         int size, float alpha, float beta, float k, cudaStream_t s) {
    const int cv = g.C / 8;
    if (cv > 32) return cudaErrorInvalidValue;
    const int HB = (g.H + 1) / 2, WB = (g.W + 1) / 2;
    // strips of `rows` block rows (each strip recomputes one halo window row: (rows+1)/rows LRN
    // work) split into column segments of cseg blocks (one recomputed window column each)
    int rows = g_fused_rb > 0 ? g_fused_rb : 4;
    rows = rows >= 4 ? 4 : rows >= 2 ? 2 : 1;
    if (rows > HB) rows = HB >= 2 ? 2 : 1;
    const int nstrip = (HB + rows - 1) / rows;
    const int ncseg = WB >= 16 ? 2 : 1, cseg = (WB + ncseg - 1) / ncseg;
    const int ntask = g.N * nstrip * ncseg;
    const int ppw = 32 / cv;
    const unsigned grid = warps_grid((ntask + ppw - 1) / ppw);
    const float an = alpha / size, cb = 2.f * an * beta;
    auto P = (const __nv_bfloat16*)p;
    auto DN = (const __nv_bfloat16*)dn;
    auto M = (const uint8_t*)mask;
    auto DX = (__nv_bfloat16*)dx;
    switch ((size - 1) / 2) {
        case 0: lrn_pool_bwd_r<0>(rows, relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb); break;
        case 1: lrn_pool_bwd_r<1>(rows, relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb); break;
        case 2: lrn_pool_bwd_r<2>(rows, relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb); break;
        case 3: lrn_pool_bwd_r<3>(rows, relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb); break;
        default: lrn_pool_bwd_r<4>(rows, relu, grid, s, P, DN, M, DX, g, HB, WB, nstrip, cseg, ncseg, ntask, an, beta, k, cb); break;
    }
    note_launch();
    return cudaGetLastError();
}

// ================================================================ softmax with loss
// One block of 16 warps; warp w owns rows w, w+16, ...; per-warp loss sums in row order, then a
// fixed-order sum over warps -> deterministic mean.
// One 8-CTA cluster, one warp per row (rows strided over the 8 x 16 warps); the loss is reduced in
// a fixed order -- lanes, then warps of a CTA, then the 8 CTAs read through distributed shared
// memory by rank 0 -- so it is deterministic without a workspace.
// One cluster of SOFTMAX_CTAS (16, a non-portable size) x 16 warps: one row per warp at batch 256.
#define SOFTMAX_CTAS 16
__global__ void __launch_bounds__(512, 1)
softmax_loss_kernel(const void* __restrict__ s, int sb, const int32_t* __restrict__ labels, float* __restrict__ loss,
                    void* __restrict__ diff, int db, int N, int K) {
    __shared__ float wl[32];
    __shared__ float block_sum;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int gw = (int)cluster.block_rank() * nw + warp, gnw = nw * SOFTMAX_CTAS;
    float my = 0.f;
    for (int n = gw; n < N; n += gnw) {
        const int base = n * K;
        const int lab = labels[n];
        // a label outside [0, K) is never read through: its row's loss term and diff are NaN
        const bool ok = (unsigned)lab < (unsigned)K;
        const float bad = ok ? 0.f : __int_as_float(0x7fc00000);
        if (K <= 1024 && (K & 3) == 0 && !sb && db && ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(diff)) & 15) == 0) {
            // FP32 scores, BF16 diff: lane l holds columns 4(l + 32q) .. +3 -- 16-byte loads, 8-byte
            // stores; the same arithmetic per element as below
            float v[32];
            float mx = -INFINITY;
            const float4* s4 = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(s) + base);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int k4 = lane + 32 * q;
                float4 f = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
                if (4 * k4 < K) f = __ldg(s4 + k4);
                v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
                mx = fmaxf(mx, fmaxf(fmaxf(f.x, f.y), fmaxf(f.z, f.w)));
            }
            for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            float se = 0.f;
#pragma unroll
            for (int q = 0; q < 32; q++) {
                v[q] = (4 * (lane + 32 * (q >> 2)) + (q & 3) < K) ? expf(v[q] - mx) : 0.f;
                se += v[q];
            }
            for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
            const float lse = logf(se);
            if (lane == 0) my += ok ? lse - (reinterpret_cast<const float*>(s)[base + lab] - mx) : bad;
            if (diff) {
                const float inv = 1.f / N, rse = 1.f / se;
                uint2* d2 = reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(diff) + base);
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int k4 = lane + 32 * q;
                    if (4 * k4 < K) {
                        float p[4];
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            p[e] = v[4 * q + e] * rse;
                            if (4 * k4 + e == lab) p[e] -= 1.f;
                            p[e] = p[e] * inv + bad;
                        }
                        __nv_bfloat162 h0 = __floats2bfloat162_rn(p[0], p[1]), h1 = __floats2bfloat162_rn(p[2], p[3]);
                        d2[k4] = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
                    }
                }
            }
            continue;
        }
        if (K <= 1024) {
            // the row lives in registers: one global read, one write
            float v[32];
            float mx = -INFINITY;
#pragma unroll
            for (int q = 0; q < 32; q++) {
                const int k = lane + 32 * q;
                v[q] = k < K ? ldv(s, base + k, sb) : -INFINITY;
                mx = fmaxf(mx, v[q]);
            }
            for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            float se = 0.f;
#pragma unroll
            for (int q = 0; q < 32; q++) {
                v[q] = (lane + 32 * q < K) ? expf(v[q] - mx) : 0.f;
                se += v[q];
            }
            for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
            const float lse = logf(se);
            if (lane == 0) my += ok ? lse - (ldv(s, base + lab, sb) - mx) : bad;
            if (diff) {
                const float inv = 1.f / N, rse = 1.f / se;
#pragma unroll
                for (int q = 0; q < 32; q++) {
                    const int k = lane + 32 * q;
                    if (k < K) {
                        float p = v[q] * rse;
                        if (k == lab) p -= 1.f;
                        stv(diff, base + k, db, p * inv + bad);
                    }
                }
            }
            continue;
        }
        float mx = -INFINITY;
        for (int k = lane; k < K; k += 32) mx = fmaxf(mx, ldv(s, base + k, sb));
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float se = 0.f;
        for (int k = lane; k < K; k += 32) se += expf(ldv(s, base + k, sb) - mx);
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const float lse = logf(se);
        if (lane == 0) my += ok ? lse - (ldv(s, base + lab, sb) - mx) : bad;
        if (diff) {
            const float inv = 1.f / N;
            for (int k = lane; k < K; k += 32) {
                float p = expf(ldv(s, base + k, sb) - mx - lse);
                if (k == lab) p -= 1.f;
                stv(diff, base + k, db, p * inv + bad);
            }
        }
    }
    if (lane == 0) wl[warp] = my;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < nw; w++) t += wl[w];
        block_sum = t;
    }
    cluster.sync();
    if (cluster.block_rank() == 0 && threadIdx.x == 0) {
        float t = 0.f;
        for (int r = 0; r < SOFTMAX_CTAS; r++) t += *cluster.map_shared_rank(&block_sum, r);
        *loss = t / N;
    }
    cluster.sync();   // keep every CTA's shared memory alive until rank 0 has read it
}

cudaError_t softmax_loss_k(const void* scores, int bf16, const int32_t* labels, float* loss, void* diff, int diff_bf16,
                           int N, int K, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(softmax_loss_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(SOFTMAX_CTAS);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = SOFTMAX_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, softmax_loss_kernel, scores, bf16, labels, loss, diff, diff_bf16, N, K);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

// ================================================================ SGD (R18)
// Two float4 per thread per iteration (both loaded before either is stored) so a grid of 4 blocks per
// SM keeps enough bytes in flight for HBM while leaving thread slots free for a concurrently running
// tensor-core kernel (the net overlaps each layer's update with the rest of the backward pass).
__device__ __forceinline__ void sgd4(float4& wv, const float4& gv, float4& vv, float lr, float mom, float decay,
                                     float gs) {
    sgd1(wv.x, gv.x, vv.x, lr, mom, decay, gs);
    sgd1(wv.y, gv.y, vv.y, lr, mom, decay, gs);
    sgd1(wv.z, gv.z, vv.z, lr, mom, decay, gs);
    sgd1(wv.w, gv.w, vv.w, lr, mom, decay, gs);
}
__device__ __forceinline__ uint2 bf16x4(const float4& wv) {
    __nv_bfloat162 a = __floats2bfloat162_rn(wv.x, wv.y), b = __floats2bfloat162_rn(wv.z, wv.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&a);
    pk.y = *reinterpret_cast<uint32_t*>(&b);
    return pk;
}
// <= 48 registers (launch bounds 256 x 5): a 256-thread update block then fits beside a 200-register
// tensor-core GEMM CTA (256 x 208 of the 64K registers), so the per-layer side-stream update
// co-runs with the backward GEMMs instead of delaying their launch.
__global__ void __launch_bounds__(256, 5) sgd_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ v,
                           __nv_bfloat16* __restrict__ wb, long long n, float lr, float mom, float decay, float gs) {
    const long long n4 = n / 4;
    const long long stride = (long long)gridDim.x * blockDim.x;
    float4* w4 = reinterpret_cast<float4*>(w);
    float4* v4 = reinterpret_cast<float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    uint2* b4 = reinterpret_cast<uint2*>(wb);
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; t + stride < n4; t += 2 * stride) {
        const long long u = t + stride;
        float4 wa = w4[t], wc = w4[u];
        const float4 ga = g4[t], gc = g4[u];
        float4 va = v4[t], vc = v4[u];
        sgd4(wa, ga, va, lr, mom, decay, gs);
        sgd4(wc, gc, vc, lr, mom, decay, gs);
        v4[t] = va; v4[u] = vc;
        w4[t] = wa; w4[u] = wc;
        if (wb) { b4[t] = bf16x4(wa); b4[u] = bf16x4(wc); }
    }
    for (; t < n4; t += stride) {
        float4 wa = w4[t];
        const float4 ga = g4[t];
        float4 va = v4[t];
        sgd4(wa, ga, va, lr, mom, decay, gs);
        v4[t] = va;
        w4[t] = wa;
        if (wb) b4[t] = bf16x4(wa);
    }
    for (long long q = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += stride) {
        float nw = w[q], vv = v[q];
        sgd1(nw, g[q], vv, lr, mom, decay, gs);
        v[q] = vv;
        w[q] = nw;
        if (wb) wb[q] = __float2bfloat16_rn(nw);
    }
}

int g_sgd_blocks_per_sm = 4;   // CAFFE_TUNE_SGD_BLOCKS_PER_SM
int g_sgd_threads = 256;   // CAFFE_TUNE_SGD_THREADS

cudaError_t sgd_k(float* w, const float* g, float* v, void* w_bf16, long long count, float lr, float mom, float decay,
                  float gscale, cudaStream_t s) {
    const bool al = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(w_bf16) & 7) == 0;
    if (!al) return cudaErrorMisalignedAddress;
    // prefer the maximal shared-memory carveout: an SM running update blocks can then also host a
    // tensor-core CTA (200+ KB of shared memory) without first draining to reconfigure L1/shared
    static bool carve = false;
    if (!carve) {
        cudaFuncSetAttribute(sgd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        carve = true;
    }
    const int threads = g_sgd_threads;
    const long long want = (count / 4 + 2 * threads - 1) / (2 * threads);   // blocks for 2 vectors per thread
    const int grid = (int)std::max(1LL, std::min<long long>(148LL * g_sgd_blocks_per_sm, want));
    sgd_kernel<<<grid, threads, 0, s>>>(w, g, v, (__nv_bfloat16*)w_bf16, count, lr, mom, decay, gscale);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cb
