// pack.cu -- layout kernels around the tensor-core GEMM: NCHW -> packed NHWC activations
// (with space-to-depth for strided convolutions), weight repacks for forward and data-gradient
// operands, the s2d data-gradient unpack, and the fixed-order weight-gradient split reduction.
// These are bandwidth kernels: one read and one write of each element, 16-byte stores.
#include "internal.h"

#include <cuda_bf16.h>

namespace cb {

__device__ __forceinline__ float ld_any(const void* p, long long i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

static inline unsigned blocks_for(long long n, int t) {
    long long b = (n + t - 1) / t;
    return (unsigned)(b > 0x7fffffff ? 0x7fffffff : b);
}

// ---------------------------------------------------------------- activations
// One thread = one packed pixel x 8 consecutive packed channels.  Pixel index fastest so the
// NCHW reads of a warp are consecutive w.
__global__ void pack_nhwc_kernel(const void* __restrict__ src, int src_bf16, void* __restrict__ dst, int dst_esz,
                                 PackGeom g, long long total) {
    const int Ctot = g.G * g.Cgp;
    const int cvecs = Ctot / 8;
    const long long HWp = (long long)g.Hp * g.Wp;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long pix = t % HWp;
        long long r = t / HWp;
        const int cv = (int)(r % cvecs);
        const int n = (int)(r / cvecs);
        const int Y = (int)(pix / g.Wp), X = (int)(pix % g.Wp);
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const int cpk = cv * 8 + e;
            const int grp = cpk / g.Cgp, cc = cpk % g.Cgp;
            float x = 0.f;
            if (cc < g.Cg * g.sh * g.sw) {
                const int d = cc / g.Cg, c = cc % g.Cg;
                const int dy = d / g.sw, dx = d % g.sw;
                const int h = Y * g.sh + dy - g.ph, w = X * g.sw + dx - g.pw;
                if (h >= 0 && h < g.H && w >= 0 && w < g.W)
                    x = ld_any(src, (((long long)n * g.C + grp * g.Cg + c) * g.H + h) * g.W + w, src_bf16);
            }
            v[e] = x;
        }
        const long long o = ((long long)n * HWp + pix) * Ctot + cv * 8;
        if (dst_esz == 2) {
            uint4 pk;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dst) + o) = pk;
        } else {
            float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + o);
            d4[0] = make_float4(tf32_rn(v[0]), tf32_rn(v[1]), tf32_rn(v[2]), tf32_rn(v[3]));
            d4[1] = make_float4(tf32_rn(v[4]), tf32_rn(v[5]), tf32_rn(v[6]), tf32_rn(v[7]));
        }
    }
}

cudaError_t pack_nhwc(const void* src, int src_bf16, void* dst, int dst_esz, const PackGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.Hp * g.Wp * (g.G * g.Cgp / 8);
    if (total == 0) return cudaSuccess;
    pack_nhwc_kernel<<<blocks_for(total, 256), 256, 0, s>>>(src, src_bf16, dst, dst_esz, g, total);
    return cudaGetLastError();
}

__global__ void unpack_s2d_kernel(const float* __restrict__ T, void* __restrict__ dX, int dx_bf16, float beta,
                                  PackGeom g, long long total) {
    const int Ctot = g.G * g.Cgp;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(t % g.W);
        long long r = t / g.W;
        const int h = (int)(r % g.H);
        r /= g.H;
        const int cfull = (int)(r % g.C);
        const int n = (int)(r / g.C);
        const int grp = cfull / g.Cg, c = cfull % g.Cg;
        const int hh = h + g.ph, ww = w + g.pw;
        const int Y = hh / g.sh, dy = hh % g.sh, X = ww / g.sw, dx = ww % g.sw;
        float v = 0.f;
        if (Y < g.Hp && X < g.Wp)
            v = T[(((long long)n * g.Hp + Y) * g.Wp + X) * Ctot + grp * g.Cgp + (dy * g.sw + dx) * g.Cg + c];
        if (dx_bf16) {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(dX) + t;
            if (beta != 0.f) v += beta * __bfloat162float(*o);
            *o = __float2bfloat16_rn(v);
        } else {
            float* o = reinterpret_cast<float*>(dX) + t;
            if (beta != 0.f) v += beta * *o;
            *o = v;
        }
    }
}

cudaError_t unpack_s2d_grad(const float* T, void* dX, int dx_bf16, float beta, const PackGeom& g, cudaStream_t s) {
    const long long total = (long long)g.N * g.C * g.H * g.W;
    if (total == 0) return cudaSuccess;
    unpack_s2d_kernel<<<blocks_for(total, 256), 256, 0, s>>>(T, dX, dx_bf16, beta, g, total);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- weights
__device__ __forceinline__ float w_packed(const void* w, int w_bf16, const WGeom& g, int ofull, int bi, int bj,
                                          int cc) {
    if (cc >= g.Cg * g.sh * g.sw) return 0.f;
    const int d = cc / g.Cg, c = cc % g.Cg;
    const int i = bi * g.sh + d / g.sw, j = bj * g.sw + d % g.sw;
    if (i >= g.kh || j >= g.kw) return 0.f;
    return ld_any(w, (((long long)ofull * g.Cg + c) * g.kh + i) * g.kw + j, w_bf16);
}

__device__ __forceinline__ void st_elem(void* dst, long long i, int esz, float v) {
    if (esz == 2) reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(dst)[i] = tf32_rn(v);
}

__global__ void repack_w_fwd_kernel(const void* __restrict__ w, int w_bf16, void* __restrict__ dst, int esz, WGeom g,
                                    long long total) {
    const int taps = g.khp * g.kwp;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int cc = (int)(t % g.Cgp);
        long long r = t / g.Cgp;
        const int tap = (int)(r % taps);
        const int ofull = (int)(r / taps);
        st_elem(dst, t, esz, w_packed(w, w_bf16, g, ofull, tap / g.kwp, tap % g.kwp, cc));
    }
}

cudaError_t repack_w_fwd(const void* w, int w_bf16, void* dst, int dst_esz, const WGeom& g, cudaStream_t s) {
    const long long total = (long long)g.O * g.khp * g.kwp * g.Cgp;
    repack_w_fwd_kernel<<<blocks_for(total, 256), 256, 0, s>>>(w, w_bf16, dst, dst_esz, g, total);
    return cudaGetLastError();
}

__global__ void repack_w_dgrad_kernel(const void* __restrict__ w, int w_bf16, void* __restrict__ dst, int esz,
                                      WGeom g, int Cge, long long total) {
    const int taps = g.khp * g.kwp;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int o = (int)(t % g.Ogp);
        long long r = t / g.Ogp;
        const int tap = (int)(r % taps);
        r /= taps;
        const int cc = (int)(r % Cge);
        const int grp = (int)(r / Cge);
        float v = 0.f;
        if (o < g.Og) {
            const int ip = tap / g.kwp, jp = tap % g.kwp;
            v = w_packed(w, w_bf16, g, grp * g.Og + o, g.khp - 1 - ip, g.kwp - 1 - jp, cc);
        }
        st_elem(dst, t, esz, v);
    }
}

cudaError_t repack_w_dgrad(const void* w, int w_bf16, void* dst, int dst_esz, const WGeom& g, int Cge,
                           cudaStream_t s) {
    const long long total = (long long)g.G * Cge * g.khp * g.kwp * g.Ogp;
    repack_w_dgrad_kernel<<<blocks_for(total, 256), 256, 0, s>>>(w, w_bf16, dst, dst_esz, g, Cge, total);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- wgrad split reduction
// Thread = one partial row/column (g, o, chunk q, row-in-chunk rr), rr fastest so the partial
// reads are coalesced.  Sums the splits in ascending order (deterministic), then maps the
// packed (tap, cc) back to (c, i, j) of the original filter.
__global__ void wgrad_reduce_kernel(const float* __restrict__ partial, float* __restrict__ dW, float beta, WGeom g,
                                    int m_tiles, int n_tiles, int splits, int BN, int chunk, int cblocks,
                                    int chunks_per_tile, long long total) {
    const int nq = g.khp * g.kwp * cblocks;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int rr = (int)(t % chunk);
        long long r = t / chunk;
        const int q = (int)(r % nq);
        r /= nq;
        const int o = (int)(r % g.Og);
        const int grp = (int)(r / g.Og);
        const int tap = q / cblocks;
        const int cc = (q % cblocks) * chunk + rr;
        if (cc >= g.Cg * g.sh * g.sw) continue;
        const int d = cc / g.Cg, c = cc % g.Cg;
        const int i = (tap / g.kwp) * g.sh + d / g.sw, j = (tap % g.kwp) * g.sw + d % g.sw;
        if (i >= g.kh || j >= g.kw) continue;
        const int m_tile = q / chunks_per_tile, row = (q % chunks_per_tile) * chunk + rr;
        const int n_tile = o / BN, col = o % BN;
        float acc = 0.f;
        for (int sp = 0; sp < splits; sp++) {
            const long long unit = (((long long)sp * g.G + grp) * m_tiles + m_tile) * n_tiles + n_tile;
            acc += partial[(unit * BN + col) * 128 + row];
        }
        float* p = dW + (((long long)(grp * g.Og + o) * g.Cg + c) * g.kh + i) * g.kw + j;
        *p = (beta != 0.f ? beta * *p : 0.f) + acc;
    }
}

cudaError_t wgrad_reduce(const float* partial, float* dW, float beta, const WGeom& g, int m_tiles, int n_tiles,
                         int splits, int BN, int chunk, int cblocks, cudaStream_t s) {
    const long long total = (long long)g.G * g.Og * g.khp * g.kwp * cblocks * chunk;
    wgrad_reduce_kernel<<<blocks_for(total, 256), 256, 0, s>>>(partial, dW, beta, g, m_tiles, n_tiles, splits, BN,
                                                               chunk, cblocks, 128 / chunk, total);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- generic convert + pad
__global__ void convert_pad_kernel(const void* __restrict__ src, int src_bf16, long long ld_src, void* __restrict__ dst,
                                   int esz, long long ld_dst, long long cols, long long total) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long c = t % ld_dst, r = t / ld_dst;
        const float v = c < cols ? ld_any(src, r * ld_src + c, src_bf16) : 0.f;
        st_elem(dst, t, esz, v);
    }
}

cudaError_t convert_pad_2d(const void* src, int src_bf16, long long ld_src, void* dst, int dst_esz,
                           long long ld_dst, long long rows, long long cols, cudaStream_t s) {
    const long long total = rows * ld_dst;
    if (total == 0) return cudaSuccess;
    convert_pad_kernel<<<blocks_for(total, 256), 256, 0, s>>>(src, src_bf16, ld_src, dst, dst_esz, ld_dst, cols,
                                                               total);
    return cudaGetLastError();
}

}  // namespace cb
