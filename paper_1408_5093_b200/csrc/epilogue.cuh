// epilogue.cuh -- the strided (bias / beta / ReLU / bf16-or-fp32) tensor-core epilogue shared by
// the GEMM kernels: one thread owns one accumulator row (TMEM lane) and writes its BN columns.
#pragma once
#include "internal.h"
#include "ptx.cuh"
#include <cuda_bf16.h>

namespace cb {

// taddr: TMEM address of this warp's lanes, column 0 of the accumulator.  rbase: element offset of
// the output row; col0: first tile column (for the N bound); cbase: output channel of tile column 0;
// bs: this tile's bias staged in shared memory (or unused when args.bias == nullptr).
__device__ __forceinline__ void epi_store_strided(const TcArgs& args, uint32_t taddr, bool row_ok, long long rbase,
                                                  int col0, int cbase, const float* bs) {
    const bool rowvec = args.s_c == 1;        // channels-last / row-major output
    const bool bf = args.out_bf16 != 0;
    const float beta = args.beta;
    const int relu = args.relu;
    auto emit16 = [&](const uint32_t (&v)[16], int c0) {
        const int nvalid = min(16, args.N - (col0 + c0));
        float x[16];
#pragma unroll
        for (int j = 0; j < 16; j++) x[j] = __uint_as_float(v[j]);
        if (args.bias) {
            const float4* b4 = reinterpret_cast<const float4*>(bs + c0);
#pragma unroll
            for (int q4 = 0; q4 < 4; q4++) {
                const float4 b = b4[q4];
                x[4 * q4] += b.x; x[4 * q4 + 1] += b.y; x[4 * q4 + 2] += b.z; x[4 * q4 + 3] += b.w;
            }
        }
        const long long off0 = rbase + (long long)(cbase + c0) * args.s_c;
        if (rowvec && nvalid == 16 && (off0 & (bf ? 7 : 3)) == 0) {
            if (bf) {
                uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.out) + off0);
                if (beta != 0.f) {
                    uint4 a = o[0], b = o[1];
                    const __nv_bfloat16* ha = reinterpret_cast<const __nv_bfloat16*>(&a);
                    const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&b);
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        x[j] += beta * __bfloat162float(ha[j]);
                        x[j + 8] += beta * __bfloat162float(hb[j]);
                    }
                }
                if (relu) {
#pragma unroll
                    for (int j = 0; j < 16; j++) x[j] = x[j] > 0.f ? x[j] : 0.f;
                }
                uint4 pk[2];
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(pk);
#pragma unroll
                for (int j = 0; j < 8; j++) h2[j] = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
                o[0] = pk[0];
                o[1] = pk[1];
            } else {
                float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.out) + off0);
                if (beta != 0.f) {
#pragma unroll
                    for (int q4 = 0; q4 < 4; q4++) {
                        const float4 a = o[q4];
                        x[4 * q4] += beta * a.x; x[4 * q4 + 1] += beta * a.y;
                        x[4 * q4 + 2] += beta * a.z; x[4 * q4 + 3] += beta * a.w;
                    }
                }
                if (relu) {
#pragma unroll
                    for (int j = 0; j < 16; j++) x[j] = x[j] > 0.f ? x[j] : 0.f;
                }
#pragma unroll
                for (int q4 = 0; q4 < 4; q4++)
                    o[q4] = make_float4(x[4 * q4], x[4 * q4 + 1], x[4 * q4 + 2], x[4 * q4 + 3]);
            }
        } else {
            // column-coalesced scalar path (NCHW: the 32 lanes write 32 consecutive pixels)
            const long long sc = args.s_c;
            if (bf) {
                __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(args.out) + off0;
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    if (j < nvalid) {
                        float y = x[j];
                        if (beta != 0.f) y += beta * __bfloat162float(o[j * sc]);
                        if (relu) y = y > 0.f ? y : 0.f;
                        o[j * sc] = __float2bfloat16_rn(y);
                    }
                }
            } else {
                float* o = reinterpret_cast<float*>(args.out) + off0;
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    if (j < nvalid) {
                        float y = x[j];
                        if (beta != 0.f) y += beta * o[j * sc];
                        if (relu) y = y > 0.f ? y : 0.f;
                        o[j * sc] = y;
                    }
                }
            }
        }
    };
    // two 16-column TMEM loads in flight per wait
    for (int c0 = 0; c0 < args.BN; c0 += 32) {
        if (col0 + c0 >= args.N) break;  // warp-uniform
        const bool two = c0 + 16 < args.BN && col0 + c0 + 16 < args.N;
        uint32_t v0[16], v1[16];
        tmem_ld16(taddr + c0, v0);
        if (two) tmem_ld16(taddr + c0 + 16, v1);
        tmem_wait_ld();
        if (!row_ok) continue;
        emit16(v0, c0);
        if (two) emit16(v1, c0 + 16);
    }
}

// TMA-store form (row-major output, beta == 0): each epilogue warp stages its 32 rows x 128 bytes
// (32 FP32 or 64 BF16 columns) in a 128-byte-swizzled shared buffer -- conflict-free 16-byte
// writes -- and one lane issues a tensor store; two buffers per warp keep one store in flight.
// Full 128-byte lines reach L2 instead of 32 partial lines per warp store instruction.
// row0: output row of this warp's lane 0; ccol: output column of tile column 0; stage: 8 KB.
__device__ __forceinline__ void epi_store_tma(const TcArgs& args, const CUtensorMap* mapC, uint32_t taddr, int row0,
                                              int col0, int ccol, const float* bs, uint8_t* stage, int& buf,
                                              int lane) {
    const bool bf = args.out_bf16 != 0;
    const int cw = bf ? 64 : 32;
    for (int c0 = 0; c0 < args.BN; c0 += cw) {
        if (col0 + c0 >= args.N) break;   // warp-uniform
        uint32_t v[64];
        tmem_ld16(taddr + c0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld16(taddr + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        if (bf) {
            tmem_ld16(taddr + c0 + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
            tmem_ld16(taddr + c0 + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
        }
        tmem_wait_ld();
        float x[64];
#pragma unroll
        for (int j = 0; j < 64; j++) x[j] = __uint_as_float(v[j]);
        if (args.bias) {
#pragma unroll
            for (int j = 0; j < 64; j++)
                if (j < cw) x[j] += bs[c0 + j];
        }
        if (args.relu) {
#pragma unroll
            for (int j = 0; j < 64; j++) x[j] = x[j] > 0.f ? x[j] : 0.f;
        }
        if (lane == 0) tma_store_wait_read1();
        __syncwarp();
        uint8_t* st = stage + buf * 4096 + lane * 128;
        const int sw = lane & 7;
        if (bf) {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                uint4 pk;
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
                for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(x[8 * j + 2 * e], x[8 * j + 2 * e + 1]);
                *reinterpret_cast<uint4*>(st + ((j ^ sw) << 4)) = pk;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
                *reinterpret_cast<float4*>(st + ((j ^ sw) << 4)) =
                    make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(mapC, stage + buf * 4096, ccol + c0, row0);
            tma_store_commit();
        }
        buf ^= 1;
    }
}

// Row-staged form for channels-last / row-major outputs (s_c == 1, beta == 0): each warp stages its
// 32 rows x 128 bytes (64 BF16 or 32 FP32 columns) in a swizzled 4 KB shared buffer, then writes
// them back in 16-byte pieces where 8 consecutive lanes cover one row's 128 contiguous bytes, so
// every store instruction writes 4 whole 128-byte segments instead of 32 scattered pieces.  Any
// row mapping works (halo tiles, groups).  Bias and ReLU are applied before staging -- the values
// written are bit-identical to epi_store_strided's.  Requires N % (16/esz) == 0, 16-byte aligned
// rows and column offsets (checked by the caller).
__device__ __forceinline__ void epi_store_rows(const TcArgs& args, uint32_t taddr, bool row_ok, long long rbase,
                                               int col0, int cbase, const float* bs, uint8_t* stage, int lane) {
    const bool bf = args.out_bf16 != 0;
    const int esz = bf ? 2 : 4;
    const int cw = bf ? 64 : 32;
    const unsigned okmask = __ballot_sync(0xffffffffu, row_ok);
    const int rb_lo = (int)(rbase & 0xffffffffLL), rb_hi = (int)(rbase >> 32);
    for (int c0 = 0; c0 < args.BN; c0 += cw) {
        if (col0 + c0 >= args.N) break;   // warp-uniform
        uint32_t v[64];
        tmem_ld16(taddr + c0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld16(taddr + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        if (bf) {
            tmem_ld16(taddr + c0 + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
            tmem_ld16(taddr + c0 + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
        }
        tmem_wait_ld();
        if (okmask == 0) continue;
        float x[64];
#pragma unroll
        for (int j = 0; j < 64; j++) x[j] = __uint_as_float(v[j]);
        if (args.bias) {
#pragma unroll
            for (int j = 0; j < 64; j++)
                if (j < cw) x[j] += bs[c0 + j];
        }
        if (args.relu) {
#pragma unroll
            for (int j = 0; j < 64; j++) x[j] = x[j] > 0.f ? x[j] : 0.f;
        }
        uint8_t* st = stage + lane * 128;
        const int sw = lane & 7;
        if (bf) {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                uint4 pk;
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
                for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(x[8 * j + 2 * e], x[8 * j + 2 * e + 1]);
                *reinterpret_cast<uint4*>(st + ((j ^ sw) << 4)) = pk;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
                *reinterpret_cast<float4*>(st + ((j ^ sw) << 4)) =
                    make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
        }
        __syncwarp();
        const int nvalid = args.N - (col0 + c0);   // valid columns of this chunk (> 0)
        const int j = lane & 7;
        const bool col_ok = j * (16 / esz) < nvalid;
#pragma unroll
        for (int it = 0; it < 8; it++) {
            const int row = it * 4 + (lane >> 3);
            const long long rb = (long long)(unsigned)__shfl_sync(0xffffffffu, rb_lo, row) |
                                 ((long long)__shfl_sync(0xffffffffu, rb_hi, row) << 32);
            if (((okmask >> row) & 1u) && col_ok) {
                const uint4 val = *reinterpret_cast<const uint4*>(stage + row * 128 + ((j ^ (row & 7)) << 4));
                *reinterpret_cast<uint4*>(reinterpret_cast<char*>(args.out) + (rb + cbase + c0) * esz + j * 16) = val;
            }
        }
        __syncwarp();
    }
}

}  // namespace cb
