// simple.cu -- CUDA-core kernels: the FP32-FMA reference convolution (math mode CAFFE_MATH_FP32),
// im2col/col2im test entry points, and the bandwidth-bound neighbour layers (ReLU, max/avg pooling,
// LRN), softmax-with-loss, bias gradient and the SGD update.
// Formulas: conv S:145/S:154, pool S:163/S:172 (+R5..R8), LRN S:217/S:226 (R9), ReLU S:199/S:208,
// softmax loss S:253/S:262, SGD S:523 (R18).
#include "internal.h"

#include <cuda_bf16.h>

namespace cb {

__device__ __forceinline__ float ldv(const void* p, long long i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void stv(void* p, long long i, int bf16, float v) {
    if (bf16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(p)[i] = v;
}
static inline unsigned nblk(long long n, int t) {
    long long b = (n + t - 1) / t;
    if (b > 148LL * 64) b = 148LL * 64;
    return (unsigned)(b < 1 ? 1 : b);
}
#define GRID_STRIDE(t, total) \
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (total); t += (long long)gridDim.x * blockDim.x)

// ================================================================ FP32 reference convolution
__global__ void conv_fwd_fp32_kernel(const void* __restrict__ x, int xb, const void* __restrict__ w, int wb,
                                     const float* __restrict__ b, void* __restrict__ y, int yb, int relu, ConvGeom g,
                                     long long total) {
    const int Cg = g.C / g.G, Og = g.O / g.G;
    GRID_STRIDE(t, total) {
        const int ox = (int)(t % g.OW);
        long long r = t / g.OW;
        const int oy = (int)(r % g.OH);
        r /= g.OH;
        const int o = (int)(r % g.O);
        const int n = (int)(r / g.O);
        const int cb = (o / Og) * Cg;
        float acc = 0.f;
        for (int c = 0; c < Cg; c++)
            for (int i = 0; i < g.kh; i++) {
                const int h = oy * g.sh - g.ph + i;
                if (h < 0 || h >= g.H) continue;
                for (int j = 0; j < g.kw; j++) {
                    const int ww = ox * g.sw - g.pw + j;
                    if (ww < 0 || ww >= g.W) continue;
                    acc = fmaf(ldv(w, (((long long)o * Cg + c) * g.kh + i) * g.kw + j, wb),
                               ldv(x, (((long long)n * g.C + cb + c) * g.H + h) * g.W + ww, xb), acc);
                }
            }
        if (b) acc += b[o];
        if (relu && !(acc > 0.f)) acc = 0.f;
        stv(y, t, yb, acc);
    }
}

cudaError_t fp32_conv_fwd(const void* x, int x_bf16, const void* w, int w_bf16, const float* b, void* y, int y_bf16,
                          int relu, const ConvGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.O * g.OH * g.OW;
    conv_fwd_fp32_kernel<<<nblk(total, 256), 256, 0, s>>>(x, x_bf16, w, w_bf16, b, y, y_bf16, relu, g, total);
    return cudaGetLastError();
}

// gather form of the data gradient: dX[n,c,h,w] = sum_{o in grp(c), i, j : y=(h+ph-i)/sh, x=(w+pw-j)/sw integral}
__global__ void conv_dgrad_fp32_kernel(const void* __restrict__ dy, int dyb, const void* __restrict__ w, int wb,
                                       void* __restrict__ dx, int dxb, float beta, ConvGeom g, long long total) {
    const int Cg = g.C / g.G, Og = g.O / g.G;
    GRID_STRIDE(t, total) {
        const int ww = (int)(t % g.W);
        long long r = t / g.W;
        const int h = (int)(r % g.H);
        r /= g.H;
        const int c = (int)(r % g.C);
        const int n = (int)(r / g.C);
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
                    acc = fmaf(ldv(w, (((long long)o * Cg + cl) * g.kh + i) * g.kw + j, wb),
                               ldv(dy, (((long long)n * g.O + o) * g.OH + oy) * g.OW + ox, dyb), acc);
                }
            }
        if (beta != 0.f) acc += beta * ldv(dx, t, dxb);
        stv(dx, t, dxb, acc);
    }
}

cudaError_t fp32_conv_dgrad(const void* dy, int dy_bf16, const void* w, int w_bf16, void* dx, int dx_bf16,
                            float beta, const ConvGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.C * g.H * g.W;
    conv_dgrad_fp32_kernel<<<nblk(total, 256), 256, 0, s>>>(dy, dy_bf16, w, w_bf16, dx, dx_bf16, beta, g, total);
    return cudaGetLastError();
}

// Block per weight element; each thread sums a fixed strided subset of the (n, y, x) range, then a
// fixed-shape tree reduction -> deterministic, blocked FP32 summation (reading R13).
__global__ void conv_wgrad_fp32_kernel(const void* __restrict__ x, int xb, const void* __restrict__ dy, int dyb,
                                       float* __restrict__ dw, float beta, ConvGeom g) {
    __shared__ float red[256];
    const int Cg = g.C / g.G, Og = g.O / g.G;
    const long long widx = blockIdx.x;
    const int j = (int)(widx % g.kw);
    long long r = widx / g.kw;
    const int i = (int)(r % g.kh);
    r /= g.kh;
    const int c = (int)(r % Cg);
    const int o = (int)(r / Cg);
    const int cfull = (o / Og) * Cg + c;
    const long long P = (long long)g.OH * g.OW, tot = (long long)g.N * P;
    float acc = 0.f;
    for (long long q = threadIdx.x; q < tot; q += blockDim.x) {
        const int n = (int)(q / P);
        const int p = (int)(q % P);
        const int oy = p / g.OW, ox = p % g.OW;
        const int h = oy * g.sh - g.ph + i, ww = ox * g.sw - g.pw + j;
        if (h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
        acc = fmaf(ldv(dy, ((long long)n * g.O + o) * P + p, dyb),
                   ldv(x, (((long long)n * g.C + cfull) * g.H + h) * g.W + ww, xb), acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) dw[widx] = (beta != 0.f ? beta * dw[widx] : 0.f) + red[0];
}

cudaError_t fp32_conv_wgrad(const void* x, int x_bf16, const void* dy, int dy_bf16, float* dw, float beta,
                            const ConvGeom& g, cudaStream_t s) {
    const long long nw = (long long)g.O * (g.C / g.G) * g.kh * g.kw;
    conv_wgrad_fp32_kernel<<<(unsigned)nw, 256, 0, s>>>(x, x_bf16, dy, dy_bf16, dw, beta, g);
    return cudaGetLastError();
}

// db[o] = beta*db + sum_{n,p} dY[n,o,p]; block per o, fixed-order strided partials + tree.
__global__ void bias_grad_kernel(const void* __restrict__ dy, int dyb, float* __restrict__ db, float beta, int N,
                                 int O, long long P) {
    __shared__ float red[256];
    const int o = blockIdx.x;
    float acc = 0.f;
    const long long tot = (long long)N * P;
    for (long long q = threadIdx.x; q < tot; q += blockDim.x) {
        const long long n = q / P, p = q % P;
        acc += ldv(dy, (n * O + o) * P + p, dyb);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) db[o] = (beta != 0.f ? beta * db[o] : 0.f) + red[0];
}

cudaError_t bias_grad(const void* dy, int dy_bf16, float* db, float beta, int N, int O, long long P, cudaStream_t s) {
    bias_grad_kernel<<<O, 256, 0, s>>>(dy, dy_bf16, db, beta, N, O, P);
    return cudaGetLastError();
}

// ================================================================ im2col / col2im (bit-exact test entry points)
__global__ void im2col_kernel(const float* __restrict__ x, int n, ConvGeom g, float* __restrict__ col, long long total) {
    const long long P = (long long)g.OH * g.OW;
    GRID_STRIDE(t, total) {
        const long long p = t % P, row = t / P;
        const int j = (int)(row % g.kw);
        const int i = (int)((row / g.kw) % g.kh);
        const int c = (int)(row / ((long long)g.kw * g.kh));
        const int oy = (int)(p / g.OW), ox = (int)(p % g.OW);
        const int h = oy * g.sh - g.ph + i, w = ox * g.sw - g.pw + j;
        col[t] = (h >= 0 && h < g.H && w >= 0 && w < g.W) ? x[(((long long)n * g.C + c) * g.H + h) * g.W + w] : 0.f;
    }
}

cudaError_t im2col_k(const float* x, int n, const ConvGeom& g, float* col, cudaStream_t s) {
    const long long total = (long long)g.C * g.kh * g.kw * g.OH * g.OW;
    im2col_kernel<<<nblk(total, 256), 256, 0, s>>>(x, n, g, col, total);
    return cudaGetLastError();
}

// gather: for each (c,h,w) sum col over (y asc, x asc) -- the FP32 order fixed by the reading.
__global__ void col2im_kernel(const float* __restrict__ col, int n, ConvGeom g, float* __restrict__ dx, long long total) {
    const long long P = (long long)g.OH * g.OW;
    GRID_STRIDE(t, total) {
        const int w = (int)(t % g.W);
        const int h = (int)((t / g.W) % g.H);
        const int c = (int)(t / ((long long)g.W * g.H));
        float acc = 0.f;
        for (int oy = 0; oy < g.OH; oy++) {
            const int i = h + g.ph - oy * g.sh;
            if (i < 0 || i >= g.kh) continue;
            for (int ox = 0; ox < g.OW; ox++) {
                const int j = w + g.pw - ox * g.sw;
                if (j < 0 || j >= g.kw) continue;
                acc += col[(((long long)c * g.kh + i) * g.kw + j) * P + (long long)oy * g.OW + ox];
            }
        }
        dx[(long long)n * g.C * g.H * g.W + t] = acc;
    }
}

cudaError_t col2im_k(const float* col, int n, const ConvGeom& g, float* dx, cudaStream_t s) {
    const long long total = (long long)g.C * g.H * g.W;
    col2im_kernel<<<nblk(total, 256), 256, 0, s>>>(col, n, g, dx, total);
    return cudaGetLastError();
}

// ================================================================ ReLU (vectorised, in-place safe)
__global__ void relu_fwd_f32(const float* __restrict__ x, float* y, long long n) {
    const long long n4 = n / 4;
    GRID_STRIDE(t, n4) {
        float4 v = reinterpret_cast<const float4*>(x)[t];
        v.x = v.x > 0.f ? v.x : 0.f; v.y = v.y > 0.f ? v.y : 0.f;
        v.z = v.z > 0.f ? v.z : 0.f; v.w = v.w > 0.f ? v.w : 0.f;
        reinterpret_cast<float4*>(y)[t] = v;
    }
    GRID_STRIDE(t, n - n4 * 4) { const float v = x[n4 * 4 + t]; y[n4 * 4 + t] = v > 0.f ? v : 0.f; }
}
__global__ void relu_fwd_bf16(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* y, long long n) {
    const long long n8 = n / 8;
    const __nv_bfloat162 z = __floats2bfloat162_rn(0.f, 0.f);
    GRID_STRIDE(t, n8) {
        uint4 v = reinterpret_cast<const uint4*>(x)[t];
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int e = 0; e < 4; e++) {
            float2 f = __bfloat1622float2(h[e]);
            h[e] = __floats2bfloat162_rn(f.x > 0.f ? f.x : 0.f, f.y > 0.f ? f.y : 0.f);
        }
        (void)z;
        reinterpret_cast<uint4*>(y)[t] = v;
    }
    GRID_STRIDE(t, n - n8 * 8) {
        const float v = __bfloat162float(x[n8 * 8 + t]);
        y[n8 * 8 + t] = __float2bfloat16_rn(v > 0.f ? v : 0.f);
    }
}

cudaError_t relu_fwd(const void* x, void* y, int bf16, long long count, cudaStream_t s) {
    const int vec = bf16 ? 8 : 4;
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    if (bf16) {
        if (!aligned) return cudaErrorMisalignedAddress;
        relu_fwd_bf16<<<nblk(count / vec + 1, 256), 256, 0, s>>>((const __nv_bfloat16*)x, (__nv_bfloat16*)y, count);
    } else {
        if (!aligned) return cudaErrorMisalignedAddress;
        relu_fwd_f32<<<nblk(count / vec + 1, 256), 256, 0, s>>>((const float*)x, (float*)y, count);
    }
    return cudaGetLastError();
}

__global__ void relu_bwd_kernel(const void* __restrict__ x, const void* dy, void* dx, int xb, int db, long long n) {
    GRID_STRIDE(t, n) {
        const float xv = ldv(x, t, xb);
        const float g = ldv(dy, t, db);
        stv(dx, t, db, xv > 0.f ? g : 0.f);
    }
}

cudaError_t relu_bwd(const void* x, const void* dy, void* dx, int x_bf16, int d_bf16, long long count, cudaStream_t s) {
    relu_bwd_kernel<<<nblk(count, 256), 256, 0, s>>>(x, dy, dx, x_bf16, d_bf16, count);
    return cudaGetLastError();
}

// ================================================================ pooling
__global__ void maxpool_fwd_kernel(const void* __restrict__ x, void* __restrict__ y, int32_t* __restrict__ mask,
                                   int bf16, PoolGeom g, long long total) {
    GRID_STRIDE(t, total) {
        const int px = (int)(t % g.OW);
        long long r = t / g.OW;
        const int py = (int)(r % g.OH);
        const long long plane = r / g.OH;
        int hs = py * g.sh - g.ph, ws = px * g.sw - g.pw;
        const int he = min(hs + g.kh, g.H), we = min(ws + g.kw, g.W);
        hs = max(hs, 0);
        ws = max(ws, 0);
        const long long base = plane * g.H * g.W;
        float best = 0.f;
        int arg = -1;
        for (int h = hs; h < he; h++)
            for (int w = ws; w < we; w++) {
                const float v = ldv(x, base + (long long)h * g.W + w, bf16);
                if (arg < 0 || v > best) { best = v; arg = h * g.W + w; }
            }
        stv(y, t, bf16, best);
        if (mask) mask[t] = arg;
    }
}

cudaError_t maxpool_fwd(const void* x, void* y, int32_t* mask, int bf16, const PoolGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.C * g.OH * g.OW;
    maxpool_fwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, y, mask, bf16, g, total);
    return cudaGetLastError();
}

// gather per input element over the windows that may contain it, ascending (py, px) -- R8, bit-exact.
__global__ void maxpool_bwd_kernel(const void* __restrict__ dy, const int32_t* __restrict__ mask, void* __restrict__ dx,
                                   int bf16, PoolGeom g, long long total) {
    GRID_STRIDE(t, total) {
        const int w = (int)(t % g.W);
        long long r = t / g.W;
        const int h = (int)(r % g.H);
        const long long plane = r / g.H;
        const int py0 = max(0, (h + g.ph - g.kh + g.sh) / g.sh), py1 = min(g.OH - 1, (h + g.ph) / g.sh);
        const int px0 = max(0, (w + g.pw - g.kw + g.sw) / g.sw), px1 = min(g.OW - 1, (w + g.pw) / g.sw);
        const int me = h * g.W + w;
        const long long base = plane * g.OH * g.OW;
        float acc = 0.f;
        for (int py = py0; py <= py1; py++)
            for (int px = px0; px <= px1; px++) {
                const long long q = base + (long long)py * g.OW + px;
                if (mask[q] == me) acc += ldv(dy, q, bf16);
            }
        stv(dx, t, bf16, acc);
    }
}

cudaError_t maxpool_bwd(const void* dy, const int32_t* mask, void* dx, int bf16, const PoolGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.C * g.H * g.W;
    maxpool_bwd_kernel<<<nblk(total, 256), 256, 0, s>>>(dy, mask, dx, bf16, g, total);
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

__global__ void avepool_fwd_kernel(const void* __restrict__ x, void* __restrict__ y, int bf16, PoolGeom g, long long total) {
    GRID_STRIDE(t, total) {
        const int px = (int)(t % g.OW);
        long long r = t / g.OW;
        const int py = (int)(r % g.OH);
        const long long plane = r / g.OH;
        int hs, he, ws, we, size;
        ave_window(py, px, g, hs, he, ws, we, size);
        float acc = 0.f;
        for (int h = hs; h < he; h++)
            for (int w = ws; w < we; w++) acc += ldv(x, plane * g.H * g.W + (long long)h * g.W + w, bf16);
        stv(y, t, bf16, acc / size);
    }
}

cudaError_t avepool_fwd(const void* x, void* y, int bf16, const PoolGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.C * g.OH * g.OW;
    avepool_fwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, y, bf16, g, total);
    return cudaGetLastError();
}

__global__ void avepool_bwd_kernel(const void* __restrict__ dy, void* __restrict__ dx, int bf16, PoolGeom g, long long total) {
    GRID_STRIDE(t, total) {
        const int w = (int)(t % g.W);
        long long r = t / g.W;
        const int h = (int)(r % g.H);
        const long long plane = r / g.H;
        const int py0 = max(0, (h + g.ph - g.kh + g.sh) / g.sh), py1 = min(g.OH - 1, (h + g.ph) / g.sh);
        const int px0 = max(0, (w + g.pw - g.kw + g.sw) / g.sw), px1 = min(g.OW - 1, (w + g.pw) / g.sw);
        float acc = 0.f;
        for (int py = py0; py <= py1; py++)
            for (int px = px0; px <= px1; px++) {
                int hs, he, ws, we, size;
                ave_window(py, px, g, hs, he, ws, we, size);
                if (h >= hs && h < he && w >= ws && w < we)
                    acc += ldv(dy, plane * g.OH * g.OW + (long long)py * g.OW + px, bf16) / size;
            }
        stv(dx, t, bf16, acc);
    }
}

cudaError_t avepool_bwd(const void* dy, void* dx, int bf16, const PoolGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.C * g.H * g.W;
    avepool_bwd_kernel<<<nblk(total, 256), 256, 0, s>>>(dy, dx, bf16, g, total);
    return cudaGetLastError();
}

// ================================================================ LRN across channels
__device__ __forceinline__ float lrn_scale(const void* x, int bf16, long long base, long long P, int c, int C, int r,
                                           float alpha_n, float k) {
    float s = 0.f;
    const int lo = max(0, c - r), hi = min(C - 1, c + r);
    for (int cc = lo; cc <= hi; cc++) {
        const float v = ldv(x, base + cc * P, bf16);
        s = fmaf(v, v, s);
    }
    return k + alpha_n * s;
}

__global__ void lrn_fwd_kernel(const void* __restrict__ x, void* __restrict__ y, float* __restrict__ scale, int bf16,
                               int C, long long P, int size, float alpha, float beta, float k, long long total) {
    const int r = (size - 1) / 2;
    const float an = alpha / size;
    GRID_STRIDE(t, total) {
        const long long p = t % P;
        const long long nc = t / P;
        const int c = (int)(nc % C);
        const long long base = (nc - c) * P + p;
        const float S = lrn_scale(x, bf16, base, P, c, C, r, an, k);
        stv(y, t, bf16, ldv(x, t, bf16) * exp2f(-beta * log2f(S)));
        if (scale) scale[t] = S;
    }
}

cudaError_t lrn_fwd(const void* x, void* y, float* scale, int bf16, int N, int C, long long P, int size, float alpha,
                    float beta, float k, cudaStream_t s) {
    const long long total = (long long)N * C * P;
    lrn_fwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, y, scale, bf16, C, P, size, alpha, beta, k, total);
    return cudaGetLastError();
}

__global__ void lrn_bwd_kernel(const void* __restrict__ x, const void* __restrict__ y, const void* __restrict__ dy,
                               const float* __restrict__ scale, void* __restrict__ dx, int bf16, int C, long long P,
                               int size, float alpha, float beta, float k, long long total) {
    const int r = (size - 1) / 2;
    const float an = alpha / size;
    GRID_STRIDE(t, total) {
        const long long p = t % P;
        const long long nc = t / P;
        const int c = (int)(nc % C);
        const long long base = (nc - c) * P + p;
        const float Sc = scale ? scale[t] : lrn_scale(x, bf16, base, P, c, C, r, an, k);
        float acc = 0.f;
        const int lo = max(0, c - r), hi = min(C - 1, c + r);
        for (int cc = lo; cc <= hi; cc++) {
            const long long q = base + cc * P;
            const float S = scale ? scale[q] : lrn_scale(x, bf16, base, P, cc, C, r, an, k);
            acc += ldv(dy, q, bf16) * ldv(y, q, bf16) / S;
        }
        const float v = ldv(dy, t, bf16) * exp2f(-beta * log2f(Sc)) - 2.f * an * beta * ldv(x, t, bf16) * acc;
        stv(dx, t, bf16, v);
    }
}

cudaError_t lrn_bwd(const void* x, const void* y, const void* dy, const float* scale, void* dx, int bf16, int N, int C,
                    long long P, int size, float alpha, float beta, float k, cudaStream_t s) {
    const long long total = (long long)N * C * P;
    lrn_bwd_kernel<<<nblk(total, 256), 256, 0, s>>>(x, y, dy, scale, dx, bf16, C, P, size, alpha, beta, k, total);
    return cudaGetLastError();
}

// ================================================================ softmax with loss
// One block of 32 warps; warp w owns rows w, w+32, ...; per-warp loss sums in row order, then a
// fixed-order sum over warps -> deterministic mean.
__global__ void softmax_loss_kernel(const void* __restrict__ s, int sb, const int32_t* __restrict__ labels,
                                    float* __restrict__ loss, void* __restrict__ diff, int db, int N, int K) {
    __shared__ float wl[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float my = 0.f;
    for (int n = warp; n < N; n += 32) {
        const long long base = (long long)n * K;
        float mx = -INFINITY;
        for (int k = lane; k < K; k += 32) mx = fmaxf(mx, ldv(s, base + k, sb));
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float se = 0.f;
        for (int k = lane; k < K; k += 32) se += expf(ldv(s, base + k, sb) - mx);
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const float lse = logf(se);
        const int lab = labels[n];
        if (lane == 0) my += lse - (ldv(s, base + lab, sb) - mx);
        if (diff) {
            const float inv = 1.f / N;
            for (int k = lane; k < K; k += 32) {
                float p = expf(ldv(s, base + k, sb) - mx - lse);
                if (k == lab) p -= 1.f;
                stv(diff, base + k, db, p * inv);
            }
        }
    }
    if (lane == 0) wl[warp] = my;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < 32; w++) t += wl[w];
        *loss = t / N;
    }
}

cudaError_t softmax_loss_k(const void* scores, int bf16, const int32_t* labels, float* loss, void* diff, int diff_bf16,
                           int N, int K, cudaStream_t s) {
    softmax_loss_kernel<<<1, 1024, 0, s>>>(scores, bf16, labels, loss, diff, diff_bf16, N, K);
    return cudaGetLastError();
}

// ================================================================ SGD (R18)
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ v,
                           __nv_bfloat16* __restrict__ wb, long long n, float lr, float mom, float decay, float gs) {
    GRID_STRIDE(t, n) {
        const float wv = w[t];
        const float gp = g[t] * gs + decay * wv;
        const float vv = mom * v[t] - lr * gp;
        const float nw = wv + vv;
        v[t] = vv;
        w[t] = nw;
        if (wb) wb[t] = __float2bfloat16_rn(nw);
    }
}

cudaError_t sgd_k(float* w, const float* g, float* v, void* w_bf16, long long count, float lr, float mom, float decay,
                  float gscale, cudaStream_t s) {
    sgd_kernel<<<nblk(count, 256), 256, 0, s>>>(w, g, v, (__nv_bfloat16*)w_bf16, count, lr, mom, decay, gscale);
    return cudaGetLastError();
}

}  // namespace cb
