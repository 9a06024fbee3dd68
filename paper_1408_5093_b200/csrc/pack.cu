#include <algorithm>
// pack.cu -- layout kernels around the tensor-core GEMM: activations into the packed channels-last
// operand layout (transpose of NCHW blobs, space-to-depth for strided convolutions, dtype
// conversion), weight repacks for the forward and data-gradient operands, the s2d data-gradient
// unpack, the fixed-order weight-gradient split reduction and a generic 2-D convert/pad.
// Bandwidth kernels: one read and one write per element, 16-byte stores.
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
    if (b > 148LL * 32) b = 148LL * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------- activations
// Generic: one thread = one packed pixel x one 16-byte vector of packed channels; pixel fastest so
// NCHW reads of a warp are consecutive w.  Handles s2d, any source layout, any dtype.
__global__ void pack_generic_kernel(const void* __restrict__ src, int src_bf16, L4 ls, void* __restrict__ dst,
                                    int dst_esz, PackGeom g, int total, int cvec_fastest) {
    const int vec = 16 / dst_esz;
    const int cvecs = g.Ctot / vec;
    const int HWp = g.Hp * g.Wp;
    const int real = g.Cg * g.sh * g.sw;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        int pix, cv, n;
        if (cvec_fastest) {   // channels-last source: neighbouring threads read neighbouring channels
            cv = t % cvecs;
            const int r = t / cvecs;
            pix = r % HWp;
            n = r / HWp;
        } else {              // NCHW source: neighbouring threads read neighbouring pixels
            pix = t % HWp;
            const int r = t / HWp;
            cv = r % cvecs;
            n = r / cvecs;
        }
        const int Y = pix / g.Wp, X = pix - (pix / g.Wp) * g.Wp;
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            v[e] = 0.f;
            if (e < vec) {
                const int cpk = cv * vec + e;
                const int grp = cpk / g.cpg, cc = cpk - grp * g.cpg;
                if (cc < real && grp < g.G) {
                    const int d = cc / g.Cg, c = cc - d * g.Cg;
                    const int dy = d / g.sw, dx = d - dy * g.sw;
                    const int h = Y * g.sh + dy - g.ph, w = X * g.sw + dx - g.pw;
                    if (h >= 0 && h < g.H && w >= 0 && w < g.W)
                        v[e] = ld_any(src, (long long)n * ls.sn + (grp * g.Cg + c) * ls.sc + h * ls.sh + w * ls.sw,
                                      src_bf16);
                }
            }
        }
        const long long o = ((long long)n * HWp + pix) * g.Ctot + cv * vec;
        if (dst_esz == 2) {
            uint4 pk;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dst) + o) = pk;
        } else {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + o) =
                make_float4(tf32_rn(v[0]), tf32_rn(v[1]), tf32_rn(v[2]), tf32_rn(v[3]));
        }
    }
}

// Fast path for a stride-1 NCHW source into bf16 NHWC with natural (unpadded, cpg == Cg) channels:
// a 64-channel x 64-pixel tile is read coalesced along pixels into shared memory and written
// coalesced along channels.
__global__ void pack_transpose_kernel(const void* __restrict__ src, int src_bf16, __nv_bfloat16* __restrict__ dst,
                                      int C, int P, int Ctot) {
    __shared__ float tile[64][65];
    const int n = blockIdx.z, p0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
    const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 256 threads: 64 x 4
    const long long sbase = (long long)n * C * P;
    for (int r = ty; r < 64; r += 4) {
        const int c = c0 + r, p = p0 + tx;
        tile[r][tx] = (c < C && p < P) ? ld_any(src, sbase + (long long)c * P + p, src_bf16) : 0.f;
    }
    __syncthreads();
    // write: each thread stores 2 consecutive channels (bf16x2) of one pixel
    const int cpair = threadIdx.x & 31, prow = threadIdx.x >> 5;  // 32 pairs x 8 pixel rows
    for (int r = prow; r < 64; r += 8) {
        const int p = p0 + r, c = c0 + 2 * cpair;
        if (p < P && c < Ctot) {
            __nv_bfloat162 v = __floats2bfloat162_rn(tile[2 * cpair][r], tile[2 * cpair + 1][r]);
            if (c + 1 < Ctot)
                *reinterpret_cast<__nv_bfloat162*>(dst + ((long long)n * P + p) * Ctot + c) = v;
            else
                dst[((long long)n * P + p) * Ctot + c] = v.x;
        }
    }
}

// Space-to-depth into bf16: one thread builds one packed pixel row (all Ctot channels) with
// incremental (division-free) channel bookkeeping, writing 16-byte vectors.
__global__ void pack_s2d_kernel(const void* __restrict__ src, int src_bf16, L4 ls, __nv_bfloat16* __restrict__ dst,
                                PackGeom g, int total) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int X = t % g.Wp;
        const int r = t / g.Wp;
        const int Y = r % g.Hp;
        const int n = r / g.Hp;
        __nv_bfloat16* out = dst + (long long)t * g.Ctot;
        const long long sb = (long long)n * ls.sn;
        for (int grp = 0; grp < g.G; grp++) {
            float v[8];
            int e = 0;
            int cc = 0;
            auto flush = [&](int upto) {
                for (int q = e; q < 8; q++) v[q] = 0.f;
                uint4 pk;
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
                for (int q = 0; q < 4; q++) h2[q] = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
                *reinterpret_cast<uint4*>(out + grp * g.cpg + upto) = pk;
                e = 0;
            };
            for (int dy = 0; dy < g.sh; dy++) {
                const int h = Y * g.sh + dy - g.ph;
                for (int dx = 0; dx < g.sw; dx++) {
                    const int w = X * g.sw + dx - g.pw;
                    const bool in = h >= 0 && h < g.H && w >= 0 && w < g.W;
                    const long long pb = sb + (long long)h * ls.sh + (long long)w * ls.sw + (long long)grp * g.Cg * ls.sc;
                    for (int c = 0; c < g.Cg; c++) {
                        v[e++] = in ? ld_any(src, pb + (long long)c * ls.sc, src_bf16) : 0.f;
                        cc++;
                        if (e == 8) flush(cc - 8);
                    }
                }
            }
            // zero tail up to cpg
            while (cc < g.cpg) {
                v[e++] = 0.f;
                cc++;
                if (e == 8) flush(cc - 8);
            }
        }
    }
}

// Space-to-depth of a channels-last BF16 source (the first conv layer's image batch).  One block
// per packed row (n, Y): the sh source rows it needs are contiguous in NHWC, so they are copied
// into shared memory with aligned 16-byte loads (enough bytes in flight to cover DRAM latency);
// the packed row is then assembled as 16-byte vectors through a per-block table mapping packed
// channel -> (dy, dx, source channel).  Packed channel (dy*sw + dx)*Cg + c of pixel (Y, X) of
// group grp is X[n][grp*Cg + c][Y*sh + dy - ph][X*sw + dx - pw] (0 outside the image).
__global__ void pack_s2d_rows_kernel(const __nv_bfloat16* __restrict__ src, L4 ls, __nv_bfloat16* __restrict__ dst,
                                     PackGeom g) {
    extern __shared__ uint4 sraw[];
    const int WC = g.W * g.C;
    const int row = blockIdx.x;
    const int n = row / g.Hp, Y = row - n * g.Hp;
    const int h0 = Y * g.sh - g.ph;
    const int ha = max(h0, 0), hb = min(h0 + g.sh, g.H);           // valid source rows [ha, hb)
    const int nrows = hb > ha ? hb - ha : 0;
    const long long e0 = (long long)n * ls.sn + (long long)ha * WC; // first element (NHWC: rows contiguous)
    const unsigned long long b0 = reinterpret_cast<unsigned long long>(src + e0);
    const unsigned long long a0 = b0 & ~15ull;
    const int head = (int)(b0 - a0);                                // bytes before the first element
    const int nvec = (head + nrows * WC * 2 + 15) / 16;
    int* tab = reinterpret_cast<int*>(sraw + ((g.sh * WC * 2 + 16 + 15) / 16 + 1));
    const uint4* gsrc = reinterpret_cast<const uint4*>(a0);
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) sraw[i] = gsrc[i];
    const int real = g.Cg * g.sh * g.sw;
    for (int c = threadIdx.x; c < g.Ctot; c += blockDim.x) {
        const int grp = c / g.cpg, cc = c - grp * g.cpg;
        int e = -1;
        if (cc < real && grp < g.G) {
            const int d = cc / g.Cg, ch = cc - d * g.Cg;
            const int dy = d / g.sw, dx = d - dy * g.sw;
            e = (dy << 24) | (dx << 16) | (grp * g.Cg + ch);
        }
        tab[c] = e;
    }
    __syncthreads();
    const uint16_t* sel = reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(sraw) + head);
    const int cvecs = g.Ctot / 8;
    uint4* out = reinterpret_cast<uint4*>(dst + (long long)row * g.Wp * g.Ctot);
    for (int v = threadIdx.x; v < g.Wp * cvecs; v += blockDim.x) {
        const int X = v / cvecs, cv = v - X * cvecs;
        uint32_t hv[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int e = tab[cv * 8 + q];
            hv[q] = 0;
            if (e >= 0) {
                const int h = h0 + (e >> 24), w = X * g.sw - g.pw + ((e >> 16) & 0xff);
                if (h >= ha && h < hb && w >= 0 && w < g.W) hv[q] = sel[(h - ha) * WC + w * g.C + (e & 0xffff)];
            }
        }
        out[v] = make_uint4(hv[0] | (hv[1] << 16), hv[2] | (hv[3] << 16), hv[4] | (hv[5] << 16), hv[6] | (hv[7] << 16));
    }
}

// Space-to-depth of a channels-last BF16 image batch without padding, one group (conv1: 3
// channels, 4x4 blocks).  Packed channels [dy*sw*C, (dy+1)*sw*C) of packed pixel (Y, X) are the
// sw*C consecutive source elements of row Y*sh + dy starting at column X*sw -- one contiguous
// segment.  Thread = one (n, Y, X, dy) segment of NW 32-bit words: the covering source words are
// loaded 4-byte aligned (NHWC rows of 3 channels are only 2-byte aligned) and realigned with a
// byte permute, stored as 8-byte words; the dy = sh-1 thread also zero-fills the channel padding.
// Source elements past the image (last block column / row) are 0.  ~20 instructions per 24-byte
// segment instead of the row-staged kernel's table lookups per element.
template <int NW>
__global__ void pack_s2d_seg_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst, PackGeom g,
                                    int total) {
    constexpr int L = 2 * NW;   // elements per segment (= sw * C)
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int dy = t % g.sh;
        int r = t / g.sh;
        const int X = r % g.Wp; r /= g.Wp;
        const int Y = r % g.Hp;
        const int n = r / g.Hp;
        const int h = Y * g.sh + dy;
        const int nv = h < g.H ? max(0, min(L, (g.W - X * g.sw) * g.C)) : 0;   // valid elements
        uint32_t o[NW];
        if (nv > 0) {
            const __nv_bfloat16* p = src + (((long long)n * g.H + h) * g.W + (long long)X * g.sw) * g.C;
            const uintptr_t b = reinterpret_cast<uintptr_t>(p);
            const uint32_t* wp = reinterpret_cast<const uint32_t*>(b & ~uintptr_t(3));
            if ((b & 3) == 0) {
#pragma unroll
                for (int i = 0; i < NW; i++) o[i] = 2 * i < nv ? __ldg(wp + i) : 0u;
            } else {   // element k sits in word (k + 1) / 2
                uint32_t w[NW + 1];
#pragma unroll
                for (int j = 0; j <= NW; j++) w[j] = 2 * j - 1 < nv ? __ldg(wp + j) : 0u;
#pragma unroll
                for (int i = 0; i < NW; i++) o[i] = __byte_perm(w[i], w[i + 1], 0x5432);
            }
            if (nv < L) {   // clear the elements past the image edge
#pragma unroll
                for (int i = 0; i < NW; i++) {
                    if (2 * i >= nv) o[i] = 0u;
                    else if (2 * i + 1 >= nv) o[i] &= 0xffffu;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < NW; i++) o[i] = 0u;
        }
        __nv_bfloat16* q = dst + (((long long)n * g.Hp + Y) * g.Wp + X) * g.Ctot + dy * L;
        uint2* q2 = reinterpret_cast<uint2*>(q);
#pragma unroll
        for (int i = 0; i < NW / 2; i++) q2[i] = make_uint2(o[2 * i], o[2 * i + 1]);
        if (dy == g.sh - 1) {
            __nv_bfloat16* z = q + L;   // channels [sh*L, Ctot)
            for (int c = 0; c < g.Ctot - g.sh * L; c += 4) *reinterpret_cast<uint2*>(z + c) = make_uint2(0u, 0u);
        }
    }
}

// Channels-last FP32 activation whose packed TF32 operand has the same layout (stride 1, no padding,
// every group's channel count a multiple of 4): a TF32-RN rounding copy in 16-byte vectors.
__global__ void pack_copy_tf32_kernel(const float4* __restrict__ src, float4* __restrict__ dst, long long n4) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n4; t += (long long)gridDim.x * blockDim.x) {
        const float4 v = src[t];
        dst[t] = make_float4(tf32_rn(v.x), tf32_rn(v.y), tf32_rn(v.z), tf32_rn(v.w));
    }
}

cudaError_t pack_act(const void* src, int src_bf16, L4 ls, int src_nhwc, void* dst, int dst_esz, const PackGeom& g,
                     cudaStream_t s) {
    const bool plain = g.sh == 1 && g.sw == 1 && g.ph == 0 && g.pw == 0 && g.Hp == g.H && g.Wp == g.W;
    if (!plain && dst_esz == 2 && src_bf16 && src_nhwc && ls.sc == 1 && ls.sw == g.C && g.G == 1 && g.ph == 0 &&
        g.pw == 0 && g.sw * g.C == 12 && g.cpg == g.Ctot && g.Ctot % 8 == 0 && g.Ctot >= g.sh * 12 &&
        (g.Ctot - g.sh * 12) % 4 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 &&
        ls.sn == (long long)g.H * g.W * g.C) {
        const int total = g.N * g.Hp * g.Wp * g.sh;
        pack_s2d_seg_kernel<6><<<blocks_for(total, 256), 256, 0, s>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst, g,
                                                                       total);
        note_launch();
        return cudaGetLastError();
    }
    if (plain && dst_esz == 4 && !src_bf16 && src_nhwc && ls.sc == 1 && g.cpg == g.Cg && g.G * g.Cg == g.C &&
        g.Ctot == g.C && g.C % 4 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 &&
        ls.sw == g.C && ls.sh == (long long)g.W * g.C && ls.sn == (long long)g.H * g.W * g.C) {
        const long long n4 = (long long)g.N * g.H * g.W * g.C / 4;
        const long long want = (n4 + 255) / 256;
        pack_copy_tf32_kernel<<<(unsigned)std::min<long long>(want, 148LL * 16), 256, 0, s>>>(
            (const float4*)src, (float4*)dst, n4);
        note_launch();
        return cudaGetLastError();
    }
    const size_t rows_smem = ((size_t)g.sh * g.W * g.C * 2 + 16 + 15) / 16 * 16 + 16 + (size_t)g.Ctot * 4;
    if (!plain && dst_esz == 2 && src_bf16 && src_nhwc && ls.sc == 1 && ls.sw == g.C && g.Ctot % 8 == 0 &&
        rows_smem <= 96 * 1024 && g.C < 65536 && g.sh < 128 && g.sw < 256) {
        static bool attr_set = false;
        if (!attr_set) {
            cudaFuncSetAttribute(pack_s2d_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            attr_set = true;
        }
        pack_s2d_rows_kernel<<<g.N * g.Hp, 128, rows_smem, s>>>((const __nv_bfloat16*)src, ls, (__nv_bfloat16*)dst, g);
    } else if (!plain && dst_esz == 2 && g.cpg % 8 == 0) {
        const int total = g.N * g.Hp * g.Wp;
        pack_s2d_kernel<<<blocks_for(total, 128), 128, 0, s>>>(src, src_bf16, ls, (__nv_bfloat16*)dst, g, total);
    } else if (plain && !src_nhwc && dst_esz == 2 && g.cpg == g.Cg && g.G * g.Cg <= g.Ctot) {
        const int P = g.H * g.W;
        dim3 grid((P + 63) / 64, (g.Ctot + 63) / 64, g.N);
        pack_transpose_kernel<<<grid, 256, 0, s>>>(src, src_bf16, (__nv_bfloat16*)dst, g.C, P, g.Ctot);
    } else {
        const int total = g.N * g.Hp * g.Wp * (g.Ctot * dst_esz / 16);
        if (total == 0) return cudaSuccess;
        pack_generic_kernel<<<blocks_for(total, 256), 256, 0, s>>>(src, src_bf16, ls, dst, dst_esz, g, total,
                                                                    src_nhwc);
    }
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- I8 image input
// Integer image batch (channels-last int8, e.g. mean-subtracted pixels) -> packed BF16 operand,
// the same space-to-depth / channel-padding layout as pack_act (exact: |v| <= 128 is a BF16).
// Segment form (one thread per (n, Y, X, dy): the sw*C contiguous bytes of one source row, L <= 16)
// with the channel padding cleared by the dy = sh-1 thread; element form otherwise.
__global__ void pack_i8_seg_kernel(const int8_t* __restrict__ src, __nv_bfloat16* __restrict__ dst, PackGeom g,
                                   int total) {
    const int L = g.sw * g.C;
    const int8_t* src_end = src + (long long)g.N * g.H * g.W * g.C;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int dy = t % g.sh;
        int r = t / g.sh;
        const int X = r % g.Wp; r /= g.Wp;
        const int Y = r % g.Hp;
        const int n = r / g.Hp;
        const int h = Y * g.sh + dy;
        const int nv = h < g.H ? max(0, min(L, (g.W - X * g.sw) * g.C)) : 0;   // valid elements
        const int8_t* p = src + (((long long)n * g.H + h) * g.W + (long long)X * g.sw) * g.C;
        uint32_t o[8];
        if (L == 12 && nv == 12 && p + 16 <= src_end) {
            // whole 12-byte segment: three (or four, when unaligned) word loads + funnel shifts
            // instead of twelve byte loads
            const uintptr_t b = reinterpret_cast<uintptr_t>(p);
            const uint32_t* wp = reinterpret_cast<const uint32_t*>(b & ~uintptr_t(3));
            const uint32_t sh = (uint32_t)(b & 3) * 8u;
            const uint32_t w0 = __ldg(wp), w1 = __ldg(wp + 1), w2 = __ldg(wp + 2);
            const uint32_t w3 = sh ? __ldg(wp + 3) : 0u;
            const uint32_t x[3] = {__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh), __funnelshift_r(w2, w3, sh)};
#pragma unroll
            for (int i = 0; i < 6; i++) {
                const float a = (float)(int8_t)(x[(2 * i) >> 2] >> (8 * ((2 * i) & 3)));
                const float c = (float)(int8_t)(x[(2 * i + 1) >> 2] >> (8 * ((2 * i + 1) & 3)));
                __nv_bfloat162 v = __floats2bfloat162_rn(a, c);
                o[i] = *reinterpret_cast<uint32_t*>(&v);
            }
            o[6] = o[7] = 0u;
        } else {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const float a = 2 * i < nv ? (float)__ldg(p + 2 * i) : 0.f;
                const float c = 2 * i + 1 < nv ? (float)__ldg(p + 2 * i + 1) : 0.f;
                __nv_bfloat162 v = __floats2bfloat162_rn(a, c);
                o[i] = *reinterpret_cast<uint32_t*>(&v);
            }
        }
        __nv_bfloat16* q = dst + (((long long)n * g.Hp + Y) * g.Wp + X) * g.Ctot + dy * L;
        if (L == 12 && (reinterpret_cast<uintptr_t>(q) & 7) == 0) {
            uint2* q2 = reinterpret_cast<uint2*>(q);
            q2[0] = make_uint2(o[0], o[1]); q2[1] = make_uint2(o[2], o[3]); q2[2] = make_uint2(o[4], o[5]);
        } else {
            uint32_t* q4 = reinterpret_cast<uint32_t*>(q);   // L even, q 4-byte aligned
#pragma unroll
            for (int i = 0; i < 8; i++)
                if (2 * i < L) q4[i] = o[i];
        }
        if (dy == g.sh - 1) {
            __nv_bfloat16* z = q + L;   // channels [sh*L, Ctot)
            for (int c = 0; c < g.Ctot - g.sh * L; c += 2) *reinterpret_cast<uint32_t*>(z + c) = 0u;
        }
    }
}
__global__ void pack_i8_generic_kernel(const int8_t* __restrict__ src, __nv_bfloat16* __restrict__ dst, PackGeom g,
                                       long long total) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(t % g.Ctot);
        long long r = t / g.Ctot;
        const int X = (int)(r % g.Wp); r /= g.Wp;
        const int Y = (int)(r % g.Hp);
        const long long n = r / g.Hp;
        const int grp = c / g.cpg, cc = c - grp * g.cpg;
        float v = 0.f;
        if (grp < g.G && cc < g.Cg * g.sh * g.sw) {
            const int d = cc / g.Cg, ch = cc - d * g.Cg;
            const int h = Y * g.sh + d / g.sw - g.ph, w = X * g.sw + d % g.sw - g.pw;
            if (h >= 0 && h < g.H && w >= 0 && w < g.W) v = (float)src[((n * g.H + h) * g.W + w) * g.C + grp * g.Cg + ch];
        }
        dst[t] = __float2bfloat16_rn(v);
    }
}

// Pixel form: one thread per packed pixel (n, Y, X) of a 4x4 space-to-depth of 3 channels (CaffeNet's
// first layer: 48 channels, no padding): its four 12-byte source segments are read as word loads +
// funnel shifts, all in flight together, and the 96-byte packed pixel leaves as six 16-byte stores
// (the segment kernel writes 8-byte pieces at a 24-byte stride, one dy row per thread).
__device__ __forceinline__ void i8_seg12(const int8_t* p, bool whole, int nv, uint32_t (&x)[3]) {
    if (whole) {
        const uintptr_t b = reinterpret_cast<uintptr_t>(p);
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(b & ~uintptr_t(3));
        const uint32_t sh = (uint32_t)(b & 3) * 8u;
        const uint32_t w0 = __ldg(wp), w1 = __ldg(wp + 1), w2 = __ldg(wp + 2);
        const uint32_t w3 = sh ? __ldg(wp + 3) : 0u;
        x[0] = __funnelshift_r(w0, w1, sh);
        x[1] = __funnelshift_r(w1, w2, sh);
        x[2] = __funnelshift_r(w2, w3, sh);
    } else {
        x[0] = x[1] = x[2] = 0u;
        for (int i = 0; i < nv; i++) x[i >> 2] |= (uint32_t)(uint8_t)__ldg(p + i) << (8 * (i & 3));
    }
}
template <bool COAL>
__global__ void __launch_bounds__(256) pack_i8_px_kernel(const int8_t* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                                         PackGeom g, int total) {
    // (a thread per 16-byte chunk, chunks fastest, measured 76 us: runtime-indexed segment words spill)
    // COAL: the warp's 32 packed pixels (3 KB, contiguous in the output) leave through a per-warp
    // shared-memory transpose as lane-contiguous 16-byte stores; warp-uniform loop
    __shared__ uint4 stg[COAL ? 8 : 1][COAL ? 32 * 6 + 1 : 1];
    const int8_t* src_end = src + (long long)g.N * g.H * g.W * 3;
    const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int stride = gridDim.x * blockDim.x;
    for (int tw = blockIdx.x * blockDim.x + (threadIdx.x & ~31); tw < total; tw += stride) {
        const int t = tw + ln;
        const bool act = t < total;
        uint32_t o[24];
#pragma unroll
        for (int k = 0; k < 24; k++) o[k] = 0u;
        if (act) {
            int r = t;
            const int X = r % g.Wp; r /= g.Wp;
            const int Y = r % g.Hp;
            const int n = r / g.Hp;
            const int nv = max(0, min(12, (g.W - X * 4) * 3));
            uint32_t x[4][3];
#pragma unroll
            for (int dy = 0; dy < 4; dy++) {
                const int h = Y * 4 + dy;
                const int8_t* p = src + (((long long)n * g.H + h) * g.W + (long long)X * 4) * 3;
                const int v = h < g.H ? nv : 0;
                i8_seg12(p, v == 12 && p + 16 <= src_end, v, x[dy]);
            }
#pragma unroll
            for (int k = 0; k < 24; k++) {   // channels 2k, 2k+1 = bytes of segment (2k)/12
                const int k0 = 2 * k, k1 = k0 + 1;
                const float a = (float)(int8_t)(x[k0 / 12][(k0 % 12) >> 2] >> (8 * ((k0 % 12) & 3)));
                const float c = (float)(int8_t)(x[k1 / 12][(k1 % 12) >> 2] >> (8 * ((k1 % 12) & 3)));
                __nv_bfloat162 bv = __floats2bfloat162_rn(a, c);
                o[k] = *reinterpret_cast<uint32_t*>(&bv);
            }
        }
        if constexpr (COAL) {
#pragma unroll
            for (int j = 0; j < 6; j++) stg[w][ln * 6 + j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
            __syncwarp();
            const int nval = min(32, total - tw);
            uint4* q = reinterpret_cast<uint4*>(dst + (long long)tw * 48);
#pragma unroll
            for (int j = 0; j < 6; j++) {
                const int c = j * 32 + ln;
                if (c < nval * 6) q[c] = stg[w][c];
            }
            __syncwarp();
        } else if (act) {
            uint4* q = reinterpret_cast<uint4*>(dst + (long long)t * 48);
#pragma unroll
            for (int j = 0; j < 6; j++) q[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        }
    }
}
int g_i8_rows = 1;   // CAFFE_TUNE_I8_ROWS

cudaError_t pack_act_i8(const void* src, void* dst, const PackGeom& g, cudaStream_t s) {
    const int L = g.sw * g.C;
    if (g_i8_rows && g.G == 1 && g.ph == 0 && g.pw == 0 && g.C == 3 && g.sh == 4 && g.sw == 4 && g.Ctot == 48 &&
        g.cpg == 48 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        const int total = g.N * g.Hp * g.Wp;
        if (g_i8_rows == 2)
            pack_i8_px_kernel<false><<<blocks_for(total, 256), 256, 0, s>>>((const int8_t*)src, (__nv_bfloat16*)dst, g, total);
        else
            pack_i8_px_kernel<true><<<blocks_for(total, 256), 256, 0, s>>>((const int8_t*)src, (__nv_bfloat16*)dst, g, total);
        note_launch();
        return cudaGetLastError();
    }
    if (g.G == 1 && g.ph == 0 && g.pw == 0 && L <= 16 && L % 2 == 0 && g.cpg == g.Ctot && g.Ctot >= g.sh * L &&
        (g.Ctot - g.sh * L) % 2 == 0 && g.Ctot % 2 == 0) {
        const int total = g.N * g.Hp * g.Wp * g.sh;
        pack_i8_seg_kernel<<<blocks_for(total, 256), 256, 0, s>>>((const int8_t*)src, (__nv_bfloat16*)dst, g, total);
    } else {
        const long long total = (long long)g.N * g.Hp * g.Wp * g.Ctot;
        pack_i8_generic_kernel<<<blocks_for(total, 256), 256, 0, s>>>((const int8_t*)src, (__nv_bfloat16*)dst, g, total);
    }
    note_launch();
    return cudaGetLastError();
}

// Inverse of the s2d packing for the data gradient, into a blob of any layout (lx), with beta.
__global__ void unpack_s2d_kernel(const float* __restrict__ T, void* __restrict__ dX, int dx_bf16, int xnhwc,
                                  float beta, PackGeom g, int total) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        int n, cfull, h, w, r = t;
        if (xnhwc) {
            cfull = r % g.C; r /= g.C;
            w = r % g.W; r /= g.W;
            h = r % g.H; n = r / g.H;
        } else {
            w = r % g.W; r /= g.W;
            h = r % g.H; r /= g.H;
            cfull = r % g.C; n = r / g.C;
        }
        const int grp = cfull / g.Cg, c = cfull - grp * g.Cg;
        const int hh = h + g.ph, ww = w + g.pw;
        const int Y = hh / g.sh, dy = hh - Y * g.sh, X = ww / g.sw, dx = ww - X * g.sw;
        float v = 0.f;
        if (Y < g.Hp && X < g.Wp)
            v = T[(((long long)n * g.Hp + Y) * g.Wp + X) * g.Ctot + grp * g.cpg + (dy * g.sw + dx) * g.Cg + c];
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

cudaError_t unpack_s2d_grad(const float* T, void* dX, int dx_bf16, int xnhwc, float beta, const PackGeom& g,
                            cudaStream_t s) {
    const int total = g.N * g.C * g.H * g.W;
    if (total == 0) return cudaSuccess;
    unpack_s2d_kernel<<<blocks_for(total, 256), 256, 0, s>>>(T, dX, dx_bf16, xnhwc, beta, g, total);
    note_launch();
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

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ void st_elem(void* dst, long long i, int esz, float v) {
    if (esz == 2) reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(dst)[i] = tf32_rn(v);
}

__global__ void repack_w_fwd_kernel(const void* __restrict__ w, int w_bf16, void* __restrict__ dst, int esz, WGeom g,
                                    int total) {
    const int taps = g.khp * g.kwp;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int cc = t % g.Cgp;
        const int r = t / g.Cgp;
        const int tap = r % taps;
        const int ofull = r / taps;
        st_elem(dst, t, esz, w_packed(w, w_bf16, g, ofull, tap / g.kwp, tap % g.kwp, cc));
    }
}

// Plain filters (no s2d) into BF16: thread = one (o, tap) x 8 consecutive packed channels, one
// 16-byte store; the index arithmetic of the element-wise kernel (several runtime divisions per
// element) made it issue-bound at ~8 us for a 1.7 MB filter.
template <typename T>
__global__ void repack_w_fwd_plain8(const T* __restrict__ w, __nv_bfloat16* __restrict__ dst, WGeom g, int total) {
    const int taps = g.kh * g.kw;
    const unsigned cv = (unsigned)g.Cgp / 8u;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int c0 = (int)((unsigned)t % cv) * 8;
        const unsigned r = (unsigned)t / cv;
        const int tap = (int)(r % (unsigned)taps);
        const int o = (int)(r / (unsigned)taps);
        const T* src = w + ((long long)o * g.Cg + c0) * taps + tap;
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; e++) v[e] = c0 + e < g.Cg ? to_f32(src[(long long)e * taps]) : 0.f;
        __nv_bfloat162 h[4];
#pragma unroll
        for (int e = 0; e < 4; e++) h[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
        *reinterpret_cast<uint4*>(dst + (long long)t * 8) = *reinterpret_cast<const uint4*>(h);
    }
}

cudaError_t repack_w_fwd(const void* w, int w_bf16, void* dst, int dst_esz, const WGeom& g, cudaStream_t s) {
    const int total = g.O * g.khp * g.kwp * g.Cgp;
    if (dst_esz == 2 && g.sh == 1 && g.sw == 1 && g.Cgp % 8 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        const int t8 = total / 8;
        if (w_bf16)
            repack_w_fwd_plain8<<<blocks_for(t8, 256), 256, 0, s>>>((const __nv_bfloat16*)w, (__nv_bfloat16*)dst, g, t8);
        else
            repack_w_fwd_plain8<<<blocks_for(t8, 256), 256, 0, s>>>((const float*)w, (__nv_bfloat16*)dst, g, t8);
        note_launch();
        return cudaGetLastError();
    }
    repack_w_fwd_kernel<<<blocks_for(total, 256), 256, 0, s>>>(w, w_bf16, dst, dst_esz, g, total);
    note_launch();
    return cudaGetLastError();
}

__global__ void repack_w_dgrad_kernel(const void* __restrict__ w, int w_bf16, void* __restrict__ dst, int esz,
                                      WGeom g, int Cge, int total) {
    const int taps = g.khp * g.kwp;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int o = t % g.Ogp;
        int r = t / g.Ogp;
        const int tap = r % taps;
        r /= taps;
        const int cc = r % Cge;
        const int grp = r / Cge;
        float v = 0.f;
        if (o < g.Og) {
            const int ip = tap / g.kwp, jp = tap % g.kwp;
            v = w_packed(w, w_bf16, g, grp * g.Og + o, g.khp - 1 - ip, g.kwp - 1 - jp, cc);
        }
        st_elem(dst, t, esz, v);
    }
}

// Plain filters into BF16: thread = one (group, c, tap') x 8 consecutive o, one 16-byte store.
template <typename T>
__global__ void repack_w_dgrad_plain8(const T* __restrict__ w, __nv_bfloat16* __restrict__ dst, WGeom g, int total) {
    const int taps = g.kh * g.kw;
    const unsigned ov = (unsigned)g.Ogp / 8u;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int o0 = (int)((unsigned)t % ov) * 8;
        unsigned r = (unsigned)t / ov;
        const int tap = (int)(r % (unsigned)taps);
        r /= (unsigned)taps;
        const int c = (int)(r % (unsigned)g.Cg);
        const int grp = (int)(r / (unsigned)g.Cg);
        const int ftap = taps - 1 - tap;   // (kh-1-i', kw-1-j')
        const T* src = w + (((long long)grp * g.Og + o0) * g.Cg + c) * taps + ftap;
        const long long os = (long long)g.Cg * taps;
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; e++) v[e] = o0 + e < g.Og ? to_f32(src[e * os]) : 0.f;
        __nv_bfloat162 h[4];
#pragma unroll
        for (int e = 0; e < 4; e++) h[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
        *reinterpret_cast<uint4*>(dst + (long long)t * 8) = *reinterpret_cast<const uint4*>(h);
    }
}

cudaError_t repack_w_dgrad(const void* w, int w_bf16, void* dst, int dst_esz, const WGeom& g, int Cge,
                           cudaStream_t s) {
    const int total = g.G * Cge * g.khp * g.kwp * g.Ogp;
    if (dst_esz == 2 && g.sh == 1 && g.sw == 1 && Cge == g.Cg && g.Ogp % 8 == 0 &&
        (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        const int t8 = total / 8;
        if (w_bf16)
            repack_w_dgrad_plain8<<<blocks_for(t8, 256), 256, 0, s>>>((const __nv_bfloat16*)w, (__nv_bfloat16*)dst, g, t8);
        else
            repack_w_dgrad_plain8<<<blocks_for(t8, 256), 256, 0, s>>>((const float*)w, (__nv_bfloat16*)dst, g, t8);
        note_launch();
        return cudaGetLastError();
    }
    repack_w_dgrad_kernel<<<blocks_for(total, 256), 256, 0, s>>>(w, w_bf16, dst, dst_esz, g, Cge, total);
    note_launch();
    return cudaGetLastError();
}

// sum_{sp = s0 .. s1-1} pp[sp * stride], added in ascending order (the fixed split order every
// reduction of this file uses); eight loads in flight before the eight adds
__device__ __forceinline__ float sum_splits_asc(const float* __restrict__ pp, long long stride, int s0, int s1) {
    float acc = 0.f;
    int sp = s0;
    for (; sp + 8 <= s1; sp += 8) {
        float a[8];
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = pp[(long long)(sp + k) * stride];
#pragma unroll
        for (int k = 0; k < 8; k++) acc += a[k];
    }
    for (; sp < s1; sp++) acc += pp[(long long)sp * stride];
    return acc;
}

// ---------------------------------------------------------------- wgrad split reduction
// Thread = one partial row/column (g, o, chunk q, row-in-chunk rr), rr fastest so the partial
// reads are coalesced.  Sums the splits in ascending order (deterministic), then maps the
// packed (tap, cc) back to (c, i, j) of the original filter.
__global__ void wgrad_reduce_kernel(const float* __restrict__ partial, float* __restrict__ dW, float beta, WGeom g,
                                    int m_tiles, int n_tiles, int splits, int BN, int chunk, int cblocks,
                                    int chunks_per_tile, int total, int cbmajor, float* __restrict__ db) {
    const int nq = g.khp * g.kwp * cblocks;
    if (db) {   // bias gradient from the ones chunk: pair (pairs-1) of channel block 0, row 64
        const int pairs = (g.khp * g.kwp + 1) / 2;
        const long long sstride = (long long)g.G * m_tiles * n_tiles * BN * 128;
        for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < g.G * g.Og; t += gridDim.x * blockDim.x) {
            const int o = t % g.Og, grp = t / g.Og;
            const int n_tile = o / BN, col = o % BN;
            const float* pp = partial + ((((long long)grp * m_tiles + (pairs - 1)) * n_tiles + n_tile) * BN + col) * 128 + 64;
            float acc = 0.f;
            for (int sp = 0; sp < splits; sp++) acc += pp[sp * sstride];
            db[t] = (beta != 0.f ? beta * db[t] : 0.f) + acc;
        }
    }
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int rr = t % chunk;
        int r = t / chunk;
        const int q = r % nq;
        r /= nq;
        const int o = r % g.Og;
        const int grp = r / g.Og;
        const int tap = q / cblocks;
        const int cc = (q % cblocks) * chunk + rr;
        if (cc >= g.Cg * g.sh * g.sw) continue;
        const int d = cc / g.Cg, c = cc % g.Cg;
        const int i = (tap / g.kwp) * g.sh + d / g.sw, j = (tap % g.kwp) * g.sw + d % g.sw;
        if (i >= g.kh || j >= g.kw) continue;
        const int pairs = (g.khp * g.kwp + 1) / 2;
        const int m_tile = cbmajor ? (q % cblocks) * pairs + tap / 2 : q / chunks_per_tile;
        const int row = cbmajor ? (tap & 1) * chunk + rr : (q % chunks_per_tile) * chunk + rr;
        const int n_tile = o / BN, col = o % BN;
        // fixed ascending-split order; loads batched 4 at a time so they are in flight together
        const long long sstride = (long long)g.G * m_tiles * n_tiles * BN * 128;
        const float* pp = partial + ((((long long)grp * m_tiles + m_tile) * n_tiles + n_tile) * BN + col) * 128 + row;
        const float acc = sum_splits_asc(pp, sstride, 0, splits);
        float* p = dW + (((long long)(grp * g.Og + o) * g.Cg + c) * g.kh + i) * g.kw + j;
        *p = (beta != 0.f ? beta * *p : 0.f) + acc;
    }
}

int g_wgrad_reduce_sg_min = 24;

// Many splits (the halo weight gradients split the pixel reduction over ~all SMs): SG threads per
// output each sum a contiguous range of splits (ascending, 4 loads in flight), and the SG range
// sums are added in ascending range order -- a fixed tree, so deterministic, with SG x the loads
// in flight of the one-thread-per-output form (which was latency-bound: ~150 dependent rounds).
// blockDim = (32, SG); lanes = consecutive outputs (coalesced partial rows).  The bias gradient
// (db) rides along as G*Og extra outputs after the weights.
template <int SG>
__global__ void wgrad_reduce_sg_kernel(const float* __restrict__ partial, float* __restrict__ dW, float beta, WGeom g,
                                       int m_tiles, int n_tiles, int splits, int BN, int chunk, int cblocks,
                                       int chunks_per_tile, int total, int cbmajor, float* __restrict__ db) {
    __shared__ float part[SG][33];
    const int nq = g.khp * g.kwp * cblocks;
    const int pairs = (g.khp * g.kwp + 1) / 2;
    const long long sstride = (long long)g.G * m_tiles * n_tiles * BN * 128;
    const int per = (splits + SG - 1) / SG;
    const int sp0 = min(splits, (int)threadIdx.y * per), sp1 = min(splits, sp0 + per);
    const int nout = total + (db ? g.G * g.Og : 0);
    for (int base = blockIdx.x * 32; base < nout; base += gridDim.x * 32) {
        const int t = base + threadIdx.x;
        const float* pp = nullptr;
        float* dst = nullptr;
        if (t < total) {
            const int rr = t % chunk;
            int r = t / chunk;
            const int q = r % nq;
            r /= nq;
            const int o = r % g.Og;
            const int grp = r / g.Og;
            const int tap = q / cblocks;
            const int cc = (q % cblocks) * chunk + rr;
            if (cc < g.Cg * g.sh * g.sw) {
                const int d = cc / g.Cg, c = cc % g.Cg;
                const int i = (tap / g.kwp) * g.sh + d / g.sw, j = (tap % g.kwp) * g.sw + d % g.sw;
                if (i < g.kh && j < g.kw) {
                    const int m_tile = cbmajor ? (q % cblocks) * pairs + tap / 2 : q / chunks_per_tile;
                    const int row = cbmajor ? (tap & 1) * chunk + rr : (q % chunks_per_tile) * chunk + rr;
                    const int n_tile = o / BN, col = o % BN;
                    pp = partial + ((((long long)grp * m_tiles + m_tile) * n_tiles + n_tile) * BN + col) * 128 + row;
                    dst = dW + (((long long)(grp * g.Og + o) * g.Cg + c) * g.kh + i) * g.kw + j;
                }
            }
        } else if (t < nout) {   // bias gradient: the ones chunk, pair (pairs-1) of channel block 0, row 64
            const int u = t - total;
            const int o = u % g.Og, grp = u / g.Og;
            const int n_tile = o / BN, col = o % BN;
            pp = partial + ((((long long)grp * m_tiles + (pairs - 1)) * n_tiles + n_tile) * BN + col) * 128 + 64;
            dst = db + u;
        }
        const float acc = pp ? sum_splits_asc(pp, sstride, sp0, sp1) : 0.f;
        part[threadIdx.y][threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.y == 0 && dst) {
            float r = part[0][threadIdx.x];
#pragma unroll
            for (int k = 1; k < SG; k++) r += part[k][threadIdx.x];
            *dst = (beta != 0.f ? beta * *dst : 0.f) + r;
        }
        __syncthreads();
    }
}

// Pair-mode (halo weight gradient, chunk 64) reduction, one block per (filter row g*Og+o, 64-channel
// block): thread (rr, tap) sums channel rr of tap `tap` over the splits (ascending -- the order of
// wgrad_reduce_kernel, so the results are bit-identical), the block gathers its 64 x kh*kw weights
// in shared memory and writes them as one contiguous run of dW[g*Og+o][c][kh][kw] (the
// one-thread-per-weight kernel scatters 4-byte stores at the kh*kw stride and spends most of its
// instructions on index divisions).  Plain (non-space-to-depth) filters; blockDim = (64, 16).
__global__ void wgrad_reduce_rows_kernel(const float* __restrict__ partial, float* __restrict__ dW, float beta,
                                         WGeom g, int m_tiles, int n_tiles, int splits, int BN, int cblocks,
                                         float* __restrict__ db) {
    extern __shared__ float rowbuf[];   // [64][kh*kw]
    const int taps = g.kh * g.kw;
    const int go = blockIdx.x / cblocks, cbk = blockIdx.x - go * cblocks;
    const int grp = go / g.Og, o = go - grp * g.Og;
    const int n_tile = o / BN, col = o - n_tile * BN;
    const int pairs = (taps + 1) / 2;
    const long long sstride = (long long)g.G * m_tiles * n_tiles * BN * 128;
    const float* base = partial + ((long long)grp * m_tiles * n_tiles + n_tile) * BN * 128 + (long long)col * 128;
    const long long mstride = (long long)n_tiles * BN * 128;   // one m_tile
    const int rr = threadIdx.x;
    const int c0 = cbk * 64, nc = min(64, g.Cg - c0);
    for (int tap = threadIdx.y; tap < taps; tap += blockDim.y) {
        if (rr >= nc) continue;
        const float* pp = base + (long long)(cbk * pairs + tap / 2) * mstride + (tap & 1) * 64 + rr;
        float acc = 0.f;
        int sp = 0;
        for (; sp + 4 <= splits; sp += 4) {
            const float a0 = pp[sp * sstride], a1 = pp[(sp + 1) * sstride], a2 = pp[(sp + 2) * sstride],
                        a3 = pp[(sp + 3) * sstride];
            acc += a0; acc += a1; acc += a2; acc += a3;
        }
        for (; sp < splits; sp++) acc += pp[sp * sstride];
        rowbuf[rr * taps + tap] = acc;
    }
    if (db && cbk == 0 && threadIdx.x == 0 && threadIdx.y == 0) {   // bias gradient: row 64 of the ones pair
        const float* pp = base + (long long)(pairs - 1) * mstride + 64;
        float acc = 0.f;
        for (int sp = 0; sp < splits; sp++) acc += pp[sp * sstride];
        db[go] = (beta != 0.f ? beta * db[go] : 0.f) + acc;
    }
    __syncthreads();
    float* out = dW + ((long long)go * g.Cg + c0) * taps;
    for (int k = threadIdx.y * 64 + threadIdx.x; k < nc * taps; k += 64 * blockDim.y)
        out[k] = (beta != 0.f ? beta * out[k] : 0.f) + rowbuf[k];
}

int g_wgrad_reduce_wide = 0;   // CAFFE_TUNE_WGRAD_REDUCE_WIDE (off: conv1 wgrad + reduce 88 -> 121 us with it)
int g_wgrad_reduce_rows = 0;   // CAFFE_TUNE_WGRAD_REDUCE_ROWS (off: 58.7 vs 52.6 us per step serialised, and its
                               // 1024-thread blocks co-schedule worse beside the side-stream GEMMs)

cudaError_t wgrad_reduce(const float* partial, float* dW, float beta, const WGeom& g, int m_tiles, int n_tiles,
                         int splits, int BN, int chunk, int cblocks, cudaStream_t s, int cbmajor, float* db) {
    const int total = g.G * g.Og * g.khp * g.kwp * cblocks * chunk;
    // plain filters (no space-to-depth), pair mode, fewer splits than the split-range threshold
    if (g_wgrad_reduce_rows && cbmajor && chunk == 64 && g.sh == 1 && g.sw == 1 && g.khp == g.kh && g.kwp == g.kw &&
        splits < g_wgrad_reduce_sg_min && g.kh * g.kw <= 64) {
        const size_t smem = (size_t)64 * g.kh * g.kw * 4;
        wgrad_reduce_rows_kernel<<<(unsigned)(g.G * g.Og * cblocks), dim3(64, 16), smem, s>>>(
            partial, dW, beta, g, m_tiles, n_tiles, splits, BN, cblocks, db);
        note_launch();
        return cudaGetLastError();
    }
    if (splits >= g_wgrad_reduce_sg_min) {
        const int nout = total + (db ? g.G * g.Og : 0);
        const unsigned nb = (unsigned)std::min<long long>((nout + 31) / 32, 148LL * 16);
        // 16/32 threads per output (a few partials each) measured slower than 8 (tools/reduce_probe.py)
        if (splits >= 96 && g_wgrad_reduce_wide)
            wgrad_reduce_sg_kernel<32><<<nb, dim3(32, 32), 0, s>>>(partial, dW, beta, g, m_tiles, n_tiles, splits, BN,
                                                                  chunk, cblocks, 128 / chunk, total, cbmajor, db);
        else if (splits >= 64 && g_wgrad_reduce_wide)
            wgrad_reduce_sg_kernel<16><<<nb, dim3(32, 16), 0, s>>>(partial, dW, beta, g, m_tiles, n_tiles, splits, BN,
                                                                  chunk, cblocks, 128 / chunk, total, cbmajor, db);
        else if (splits >= 32)
            wgrad_reduce_sg_kernel<8><<<nb, dim3(32, 8), 0, s>>>(partial, dW, beta, g, m_tiles, n_tiles, splits, BN,
                                                                chunk, cblocks, 128 / chunk, total, cbmajor, db);
        else
            wgrad_reduce_sg_kernel<4><<<nb, dim3(32, 4), 0, s>>>(partial, dW, beta, g, m_tiles, n_tiles, splits, BN,
                                                                chunk, cblocks, 128 / chunk, total, cbmajor, db);
        note_launch();
        return cudaGetLastError();
    }
    wgrad_reduce_kernel<<<blocks_for(total, 256), 256, 0, s>>>(partial, dW, beta, g, m_tiles, n_tiles, splits, BN,
                                                               chunk, cblocks, 128 / chunk, total, cbmajor, db);
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- split-K GEMM reduction
// out[m*ldo + n] = act( sum_{s asc} partial[unit(s, m_tile, n_tile)][n % BN][m % TM] + bias[n] + beta*out )
// unit = (s*m_tiles + m_tile)*n_tiles + n_tile (groups == 1).  m fastest -> coalesced partial reads.
__global__ void gemm_partial_reduce_kernel(const float* __restrict__ part, int splits, int m_tiles, int n_tiles,
                                           int BN, int TM, int M, int N, void* __restrict__ out, int obf16, long long ldo,
                                           const float* __restrict__ bias, int relu, float beta, int pC, int pHW,
                                           long long total) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int m = (int)(t % M), n = (int)(t / M);
        const int mt = m / TM, mr = m - mt * TM, nt = n / BN, nc = n - nt * BN;
        const long long sstride = (long long)m_tiles * n_tiles * BN * TM;
        const float* pp = part + (((long long)mt * n_tiles + nt) * BN + nc) * TM + mr;
        float acc = 0.f;
        int s = 0;
        for (; s + 4 <= splits; s += 4) {   // ascending order, 4 loads in flight
            const float a0 = pp[s * sstride], a1 = pp[(s + 1) * sstride], a2 = pp[(s + 2) * sstride],
                        a3 = pp[(s + 3) * sstride];
            acc += a0; acc += a1; acc += a2; acc += a3;
        }
        for (; s < splits; s++) acc += pp[s * sstride];
        if (bias) acc += bias[n];
        // pC > 0: column n = c*HW + hw of the (c,h,w) flatten lands at hw*C + c of an NHWC row
        const long long o = (long long)m * ldo + (pC > 0 ? (long long)(n % pHW) * pC + n / pHW : n);
        if (obf16) {
            __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(out) + o;
            if (beta != 0.f) acc += beta * __bfloat162float(*p);
            if (relu) acc = acc > 0.f ? acc : 0.f;
            *p = __float2bfloat16_rn(acc);
        } else {
            float* p = reinterpret_cast<float*>(out) + o;
            if (beta != 0.f) acc += beta * *p;
            if (relu) acc = acc > 0.f ? acc : 0.f;
            *p = acc;
        }
    }
}

// Vector form: one thread = one row m x 8 consecutive columns (BN % 8 == 0, N % 8 == 0, ldo % 8 == 0,
// row-major output): 8 coalesced partial loads per split, one 16-byte (bf16) / 32-byte (fp32) store.
__global__ void gemm_partial_reduce8_kernel(const float* __restrict__ part, int splits, int m_tiles, int n_tiles, int BN,
                                            int TM, int M, int N, void* __restrict__ out, int obf16, long long ldo,
                                            const float* __restrict__ bias, int relu, float beta, long long total,
                                            const void* __restrict__ mref, int mref_bf16) {
    const long long sstride = (long long)m_tiles * n_tiles * BN * TM;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int m = (int)(t % M), n0 = (int)(t / M) * 8;
        const int mt = m / TM, mr = m - mt * TM, nt = n0 / BN, nc = n0 - nt * BN;
        const float* pp = part + (((long long)mt * n_tiles + nt) * BN + nc) * TM + mr;
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; e++) acc[e] = 0.f;
        int sp = 0;
        for (; sp + 4 <= splits; sp += 4) {   // ascending split order; 32 loads in flight
            float v[4][8];
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int e = 0; e < 8; e++) v[q][e] = pp[(sp + q) * sstride + (long long)e * TM];
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] += v[q][e];
        }
        for (; sp < splits; sp++) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; e++) v[e] = pp[sp * sstride + (long long)e * TM];
#pragma unroll
            for (int e = 0; e < 8; e++) acc[e] += v[e];
        }
        if (bias) {
#pragma unroll
            for (int e = 0; e < 8; e++) acc[e] += bias[n0 + e];
        }
        const long long o = (long long)m * ldo + n0;
        if (mref) {   // the backward of the ReLU whose output (same layout as out) is mref
            if (mref_bf16) {   // 8 BF16 values, one 16-byte load (o is a multiple of 8)
                const uint4 rv = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(mref) + o);
                const uint32_t w4[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const uint16_t h = (uint16_t)(w4[e >> 1] >> ((e & 1) * 16));
                    acc[e] = ((h & 0x8000u) == 0 && (h & 0x7fffu) != 0) ? acc[e] : 0.f;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] = reinterpret_cast<const float*>(mref)[o + e] > 0.f ? acc[e] : 0.f;
            }
        }
        if (obf16) {
            uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + o);
            if (beta != 0.f) {
                const uint4 old = *p;
                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&old);
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] += beta * __bfloat162float(h[e]);
            }
            if (relu) {
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] = acc[e] > 0.f ? acc[e] : 0.f;
            }
            uint4 pk;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
            *p = pk;
        } else {
            float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + o);
            if (beta != 0.f) {
                const float4 a = p[0], b = p[1];
                acc[0] += beta * a.x; acc[1] += beta * a.y; acc[2] += beta * a.z; acc[3] += beta * a.w;
                acc[4] += beta * b.x; acc[5] += beta * b.y; acc[6] += beta * b.z; acc[7] += beta * b.w;
            }
            if (relu) {
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] = acc[e] > 0.f ? acc[e] : 0.f;
            }
            p[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            p[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        }
    }
}

// NHWC-scatter form (inner-product data gradient into a channels-last blob): one thread = row m x
// pixel hw x 8 consecutive channels c..c+7 (columns n = c*HW + hw of the (c,h,w) flatten), one
// 16-byte (bf16) / 32-byte (fp32) store.  Requires pC % 8 == 0.  32-bit index math.
__global__ void gemm_partial_reduce_nhwc8_kernel(const float* __restrict__ part, int splits, int m_tiles, int n_tiles,
                                                 int BN, int TM, int M, void* __restrict__ out, int obf16, long long ldo,
                                                 float beta, int pC, int pHW, int total) {
    const long long sstride = (long long)m_tiles * n_tiles * BN * TM;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int m = t % M;
        const int r = t / M;
        const int hw = r % pHW, c0 = (r / pHW) * 8;
        const int mt = m / TM, mr = m - mt * TM;
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; e++) acc[e] = 0.f;
        const float* pp[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            const int n = (c0 + e) * pHW + hw, nt = n / BN, nc = n - nt * BN;
            pp[e] = part + (((long long)mt * n_tiles + nt) * BN + nc) * TM + mr;
        }
        int sp = 0;
        for (; sp + 4 <= splits; sp += 4) {   // ascending split order; 32 loads in flight
            float v[4][8];
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int e = 0; e < 8; e++) v[q][e] = pp[e][(sp + q) * sstride];
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] += v[q][e];
        }
        for (; sp < splits; sp++) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; e++) v[e] = pp[e][sp * sstride];
#pragma unroll
            for (int e = 0; e < 8; e++) acc[e] += v[e];
        }
        const long long o = (long long)m * ldo + (long long)hw * pC + c0;
        if (obf16) {
            uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + o);
            if (beta != 0.f) {
                const uint4 old = *p;
                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&old);
#pragma unroll
                for (int e = 0; e < 8; e++) acc[e] += beta * __bfloat162float(h[e]);
            }
            uint4 pk;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
            *p = pk;
        } else {
            float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + o);
            if (beta != 0.f) {
                const float4 a = p[0], b = p[1];
                acc[0] += beta * a.x; acc[1] += beta * a.y; acc[2] += beta * a.z; acc[3] += beta * a.w;
                acc[4] += beta * b.x; acc[5] += beta * b.y; acc[6] += beta * b.z; acc[7] += beta * b.w;
            }
            p[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            p[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        }
    }
}

cudaError_t gemm_partial_reduce(const float* part, int splits, int m_tiles, int n_tiles, int BN, int TM, int M, int N,
                                void* out, int out_bf16, long long ldo, const float* bias, int relu, float beta, int pC,
                                int pHW, cudaStream_t s, const void* mref, int mref_bf16) {
    const long long total = (long long)M * N;
    const bool al = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    if (pC == 0 && BN % 8 == 0 && N % 8 == 0 && ldo % 8 == 0 && al) {
        gemm_partial_reduce8_kernel<<<blocks_for(total / 8, 256), 256, 0, s>>>(part, splits, m_tiles, n_tiles, BN, TM, M, N,
                                                                               out, out_bf16, ldo, bias, relu, beta,
                                                                               total / 8, mref, mref_bf16);
        note_launch();
        return cudaGetLastError();
    }
    if (mref) return cudaErrorNotSupported;   // the caller falls back to a separate ReLU-backward pass
    if (pC > 0 && pC % 8 == 0 && !bias && !relu && al && ldo % 8 == 0 && total / 8 < (1LL << 31)) {
        const int tv = (int)(total / 8);
        gemm_partial_reduce_nhwc8_kernel<<<blocks_for(tv, 256), 256, 0, s>>>(part, splits, m_tiles, n_tiles, BN, TM, M,
                                                                            out, out_bf16, ldo, beta, pC, pHW, tv);
        note_launch();
        return cudaGetLastError();
    }
    gemm_partial_reduce_kernel<<<blocks_for(total, 256), 256, 0, s>>>(part, splits, m_tiles, n_tiles, BN, TM, M, N, out,
                                                                       out_bf16, ldo, bias, relu, beta, pC, pHW, total);
    note_launch();
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
    note_launch();
    return cudaGetLastError();
}

// NHWC (N,H,W,C) -> NCHW-flattened rows (N, C*H*W) with dtype conversion and padded row length:
// used to stage an NHWC inner-product input in the (c,h,w) flatten order of S:130.
__global__ void nhwc_to_rows_kernel(const void* __restrict__ src, int src_bf16, void* __restrict__ dst, int esz,
                                    int C, int HW, long long ld, long long total) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long k = t % ld, n = t / ld;
        float v = 0.f;
        if (k < (long long)C * HW) {
            const int c = (int)(k / HW), p = (int)(k % HW);
            v = ld_any(src, (n * HW + p) * C + c, src_bf16);
        }
        st_elem(dst, t, esz, v);
    }
}

// BF16 -> BF16 rows, one block per (64-channel block, image): the block's HW x 64 channels are read
// as 16-byte vectors into shared memory (pitch 65) and leave as bf16x2 stores -- a warp writes 128
// contiguous bytes of the (c,h,w) row (the one-block-per-image form stores scalar 2-byte elements
// from 256 blocks: latency-bound, ~10 us for fc6's 4.7 MB input)
int g_rows_cb = 1;   // CAFFE_TUNE_ROWS_CB
__global__ void __launch_bounds__(256) nhwc_to_rows_cb_kernel(const __nv_bfloat16* __restrict__ src,
                                                              __nv_bfloat16* __restrict__ dst, int C, int HW) {
    extern __shared__ float tr_cb[];   // [HW][65]
    const int n = blockIdx.y, c0 = blockIdx.x * 64;
    const __nv_bfloat16* sp = src + (long long)n * C * HW + c0;
    for (int i = threadIdx.x; i < HW * 8; i += blockDim.x) {
        const int p = i >> 3, v = i & 7;
        const uint4 u = *reinterpret_cast<const uint4*>(sp + (long long)p * C + v * 8);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const float2 f = __bfloat1622float2(h[q]);
            tr_cb[p * 65 + v * 8 + 2 * q] = f.x;
            tr_cb[p * 65 + v * 8 + 2 * q + 1] = f.y;
        }
    }
    __syncthreads();
    __nv_bfloat162* dp = reinterpret_cast<__nv_bfloat162*>(dst + ((long long)n * C + c0) * HW);
    for (int k2 = threadIdx.x; k2 < 32 * HW; k2 += blockDim.x) {   // element pairs (k, k+1) of the block's rows
        const int k = 2 * k2, c = k / HW, p = k - c * HW;          // HW even: a pair never straddles channels
        dp[k2] = __floats2bfloat162_rn(tr_cb[p * 65 + c], tr_cb[(p + 1) * 65 + c]);
    }
}

// One block per image: the (HW x C) channels-last image is read coalesced into shared memory
// (padded pitch C+1) and written as the (c,h,w)-ordered row, coalesced; 32-bit index math.
__global__ void nhwc_to_rows_tiled_kernel(const void* __restrict__ src, int src_bf16, void* __restrict__ dst, int esz,
                                          int C, int HW, int ld) {
    extern __shared__ float tr_tile[];   // [HW][C + 1]
    const int n = blockIdx.x;
    const int CHW = C * HW;
    const long long sb = (long long)n * CHW;
    if (src_bf16 && C % 8 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        // 16-byte vectors (8 channels of one pixel), several in flight per thread
        const uint4* v = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(src) + sb);
#pragma unroll 4
        for (int i = threadIdx.x; i < CHW / 8; i += blockDim.x) {
            const uint4 u = v[i];
            const int e0 = i * 8, p = e0 / C, c = e0 - p * C;
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float2 f = __bfloat1622float2(h[q]);
                tr_tile[p * (C + 1) + c + 2 * q] = f.x;
                tr_tile[p * (C + 1) + c + 2 * q + 1] = f.y;
            }
        }
    } else {
#pragma unroll 4
        for (int i = threadIdx.x; i < CHW; i += blockDim.x) {
            const int p = i / C, c = i - p * C;
            tr_tile[p * (C + 1) + c] = ld_any(src, sb + i, src_bf16);
        }
    }
    __syncthreads();
    const long long db = (long long)n * ld;
#pragma unroll 4
    for (int k = threadIdx.x; k < ld; k += blockDim.x) {
        float v = 0.f;
        if (k < CHW) {
            const int c = k / HW, p = k - c * HW;
            v = tr_tile[p * (C + 1) + c];
        }
        st_elem(dst, db + k, esz, v);
    }
}

cudaError_t nhwc_to_rows(const void* src, int src_bf16, void* dst, int dst_esz, int N, int C, int HW, long long ld,
                         cudaStream_t s) {
    if (g_rows_cb && src_bf16 && dst_esz == 2 && C % 64 == 0 && HW % 2 == 0 && ld == (long long)C * HW &&
        HW * 65 * 4 <= 48 * 1024 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(dst) & 3) == 0 && ld < (1LL << 31)) {
        const size_t tile = (size_t)HW * 65 * sizeof(float);
        nhwc_to_rows_cb_kernel<<<dim3(C / 64, N), 256, tile, s>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst, C, HW);
        note_launch();
        return cudaGetLastError();
    }
    const size_t tile = (size_t)HW * (C + 1) * sizeof(float);
    if (tile <= 48 * 1024 && ld < (1LL << 31)) {
        nhwc_to_rows_tiled_kernel<<<N, 256, tile, s>>>(src, src_bf16, dst, dst_esz, C, HW, (int)ld);
        note_launch();
        return cudaGetLastError();
    }
    const long long total = (long long)N * ld;
    nhwc_to_rows_kernel<<<blocks_for(total, 256), 256, 0, s>>>(src, src_bf16, dst, dst_esz, C, HW, ld, total);
    note_launch();
    return cudaGetLastError();
}

// rows (N, C*H*W) fp32 -> blob of layout lx (for an NHWC inner-product data gradient), with beta.
__global__ void rows_to_blob_kernel(const float* __restrict__ src, long long ld, void* __restrict__ dst, int dbf16,
                                    int C, int HW, float beta, long long total) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        // dst is NHWC: t = (n*HW + p)*C + c
        const int c = (int)(t % C);
        const long long r = t / C;
        const int p = (int)(r % HW);
        const long long n = r / HW;
        float v = src[n * ld + (long long)c * HW + p];
        if (dbf16) {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(dst) + t;
            if (beta != 0.f) v += beta * __bfloat162float(*o);
            *o = __float2bfloat16_rn(v);
        } else {
            float* o = reinterpret_cast<float*>(dst) + t;
            if (beta != 0.f) v += beta * *o;
            *o = v;
        }
    }
}

cudaError_t rows_to_nhwc(const float* src, long long ld, void* dst, int dst_bf16, int N, int C, int HW, float beta,
                         cudaStream_t s) {
    const long long total = (long long)N * C * HW;
    rows_to_blob_kernel<<<blocks_for(total, 256), 256, 0, s>>>(src, ld, dst, dst_bf16, C, HW, beta, total);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cb
