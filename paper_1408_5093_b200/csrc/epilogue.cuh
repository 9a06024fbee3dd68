// epilogue.cuh -- the strided (bias / beta / ReLU / bf16-or-fp32) tensor-core epilogue shared by
// the GEMM kernels: one thread owns one accumulator row (TMEM lane) and writes its BN columns.
#pragma once
#include "internal.h"
#include "ptx.cuh"
#include <cuda_bf16.h>

namespace cb {

// Specialised channels-last BF16 epilogue for EPC columns (a multiple of 8) of one accumulator row:
// every TMEM load is issued before the single wait, bias comes from shared memory with vector
// loads, and the row's EPC*2 bytes leave as 16-byte stores.  Preconditions (host-checked): BF16
// output, unit column stride, beta == 0, no column tail, 16-byte aligned row segments.  Writes the
// same values as epi_store_strided (bias add, ReLU, RNE conversion in the same order).
template <int EPC>
__device__ __forceinline__ void epi_store_bf16_rowseg(uint32_t taddr, bool row_ok, __nv_bfloat16* dst,
                                                      uint32_t sbias_addr, bool bias, bool relu) {
    uint32_t v[EPC];
#pragma unroll
    for (int c = 0; c < EPC; c += 16) {
        if (c + 16 <= EPC) tmem_ld16p(taddr + c, v + c);
        else tmem_ld8p(taddr + c, v + c);
    }
    tmem_wait_ld();
    if (!row_ok) return;
    uint32_t pk[EPC / 2];
#pragma unroll
    for (int c = 0; c < EPC; c += 4) {
        float x0 = __uint_as_float(v[c]), x1 = __uint_as_float(v[c + 1]);
        float x2 = __uint_as_float(v[c + 2]), x3 = __uint_as_float(v[c + 3]);
        if (bias) {
            const float4 b = lds_f4(sbias_addr + 4u * c);
            x0 += b.x; x1 += b.y; x2 += b.z; x3 += b.w;
        }
        if (relu) {
            x0 = x0 > 0.f ? x0 : 0.f; x1 = x1 > 0.f ? x1 : 0.f;
            x2 = x2 > 0.f ? x2 : 0.f; x3 = x3 > 0.f ? x3 : 0.f;
        }
        __nv_bfloat162 h0 = __floats2bfloat162_rn(x0, x1), h1 = __floats2bfloat162_rn(x2, x3);
        pk[c / 2] = *reinterpret_cast<uint32_t*>(&h0);
        pk[c / 2 + 1] = *reinterpret_cast<uint32_t*>(&h1);
    }
    uint4* o = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < EPC / 8; q++) o[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
}

// Same arithmetic as epi_store_bf16_rowseg, with the stores coalesced through a per-warp shared-
// memory transpose: each lane stages its row's EPC/8 16-byte pieces (row stride an odd number of
// pieces: conflict-free), then the warp writes the 32 rows' pieces in order -- consecutive lanes
// store consecutive 16-byte pieces of a pixel's channel segment, so a store instruction covers ~6
// pixel segments instead of 32 scattered 16-byte pieces (the direct form is bound by the L1 store
// path at one piece per lane per cycle: conv1's 148.7 MB output).  Warp-collective: every lane
// calls it; rows with row_ok == false store nothing.
template <int EPC>
constexpr int coal_warp_bytes() { return 32 * ((EPC / 8) | 1) * 16; }

template <int EPC>
__device__ __forceinline__ void epi_store_bf16_rowseg_coal(uint32_t taddr, bool row_ok, __nv_bfloat16* dst,
                                                           uint32_t sbias_addr, bool bias, bool relu, uint32_t wstage,
                                                           int lane) {
    constexpr int NCH = EPC / 8;     // 16-byte pieces per row
    constexpr int STR = NCH | 1;     // staging row stride in pieces (odd)
    uint32_t v[EPC];
#pragma unroll
    for (int c = 0; c < EPC; c += 16) {
        if (c + 16 <= EPC) tmem_ld16p(taddr + c, v + c);
        else tmem_ld8p(taddr + c, v + c);
    }
    tmem_wait_ld();
    uint32_t pk[EPC / 2];
#pragma unroll
    for (int c = 0; c < EPC; c += 4) {
        float x0 = __uint_as_float(v[c]), x1 = __uint_as_float(v[c + 1]);
        float x2 = __uint_as_float(v[c + 2]), x3 = __uint_as_float(v[c + 3]);
        if (bias) {
            const float4 b = lds_f4(sbias_addr + 4u * c);
            x0 += b.x; x1 += b.y; x2 += b.z; x3 += b.w;
        }
        if (relu) {
            x0 = x0 > 0.f ? x0 : 0.f; x1 = x1 > 0.f ? x1 : 0.f;
            x2 = x2 > 0.f ? x2 : 0.f; x3 = x3 > 0.f ? x3 : 0.f;
        }
        __nv_bfloat162 h0 = __floats2bfloat162_rn(x0, x1), h1 = __floats2bfloat162_rn(x2, x3);
        pk[c / 2] = *reinterpret_cast<uint32_t*>(&h0);
        pk[c / 2 + 1] = *reinterpret_cast<uint32_t*>(&h1);
    }
    __syncwarp();   // the previous call's copy-out has finished reading the staging
#pragma unroll
    for (int q = 0; q < NCH; q++)
        sts_u4(wstage + (uint32_t)((lane * STR + q) * 16), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    __syncwarp();
    const unsigned ok = __ballot_sync(0xffffffffu, row_ok);
    const unsigned long long mine = reinterpret_cast<unsigned long long>(dst);
    // every piece read back from the staging before the first global store: the stores then issue
    // back to back instead of each waiting on its own shared-memory load
    uint4 piece[NCH];
    unsigned long long addr[NCH];
    bool st_ok[NCH];
#pragma unroll
    for (int it = 0; it < NCH; it++) {
        const int c = it * 32 + lane;
        const int p = c / NCH, k = c - p * NCH;
        addr[it] = __shfl_sync(0xffffffffu, mine, p) + 16ull * (unsigned long long)k;
        st_ok[it] = (ok >> p) & 1u;
        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(piece[it].x), "=r"(piece[it].y), "=r"(piece[it].z), "=r"(piece[it].w)
                     : "r"(wstage + (uint32_t)((p * STR + k) * 16)));
    }
#pragma unroll
    for (int it = 0; it < NCH; it++)
        if (st_ok[it])   // global-space store (a pointer rebuilt from an integer would be a generic ST)
            asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(addr[it]), "r"(piece[it].x), "r"(piece[it].y),
                         "r"(piece[it].z), "r"(piece[it].w)
                         : "memory");
}

// Same arithmetic as epi_store_bf16_rowseg, but the row's EPC columns (tile columns
// [col_begin, col_begin + EPC)) go to the shared-memory TMA staging of the tile: chunk q of cw
// channels holds box row r (= pixel) at q*chunk_bytes + r*cw*2, 16-byte piece k stored at
// k ^ swizzle(r) (the TMA SWIZZLE_{128,64,32}B pattern for cw = 64/32/16; none otherwise).
// cw_log2 = 0: one chunk per epilogue group (cw == EPC, unswizzled: an odd number of 16-byte
// pieces per row keeps the 32 lanes' stores conflict-free).
template <int EPC>
__device__ __forceinline__ void epi_stage_bf16_row(uint32_t taddr, bool row_ok, uint32_t stg, int r, int col_begin,
                                                   int cw_log2, int chunk_bytes, uint32_t sbias_addr, bool bias,
                                                   bool relu) {
    uint32_t v[EPC];
#pragma unroll
    for (int c = 0; c < EPC; c += 16) {
        if (c + 16 <= EPC) tmem_ld16p(taddr + c, v + c);
        else tmem_ld8p(taddr + c, v + c);
    }
    tmem_wait_ld();
    if (!row_ok) return;
    uint32_t pk[EPC / 2];
#pragma unroll
    for (int c = 0; c < EPC; c += 4) {
        float x0 = __uint_as_float(v[c]), x1 = __uint_as_float(v[c + 1]);
        float x2 = __uint_as_float(v[c + 2]), x3 = __uint_as_float(v[c + 3]);
        if (bias) {
            const float4 b = lds_f4(sbias_addr + 4u * c);
            x0 += b.x; x1 += b.y; x2 += b.z; x3 += b.w;
        }
        if (relu) {
            x0 = x0 > 0.f ? x0 : 0.f; x1 = x1 > 0.f ? x1 : 0.f;
            x2 = x2 > 0.f ? x2 : 0.f; x3 = x3 > 0.f ? x3 : 0.f;
        }
        __nv_bfloat162 h0 = __floats2bfloat162_rn(x0, x1), h1 = __floats2bfloat162_rn(x2, x3);
        pk[c / 2] = *reinterpret_cast<uint32_t*>(&h0);
        pk[c / 2 + 1] = *reinterpret_cast<uint32_t*>(&h1);
    }
    if (cw_log2 == 0) {
        const uint32_t row = stg + (uint32_t)(col_begin / EPC) * chunk_bytes + (uint32_t)r * (EPC * 2);
#pragma unroll
        for (int q = 0; q < EPC / 8; q++) sts_u4(row + 16u * q, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    } else {
        const int cw = 1 << cw_log2;
        const int sw = cw_log2 == 6 ? (r & 7) : cw_log2 == 5 ? ((r >> 1) & 3) : cw_log2 == 4 ? ((r >> 2) & 1) : 0;
        const uint32_t rowoff = (uint32_t)r * (uint32_t)(cw * 2);
#pragma unroll
        for (int q = 0; q < EPC / 8; q++) {
            const int c = col_begin + 8 * q;
            const int chunk = c >> cw_log2, k = (c & (cw - 1)) >> 3;
            sts_u4(stg + (uint32_t)chunk * chunk_bytes + rowoff + ((uint32_t)(k ^ sw) << 4), pk[4 * q], pk[4 * q + 1],
                   pk[4 * q + 2], pk[4 * q + 3]);
        }
    }
}

// taddr: TMEM address of this warp's lanes, column 0 of the accumulator.  rbase: element offset of
// the output row; col0: first tile column (for the N bound); cbase: output channel of tile column 0;
// bs: this tile's bias staged in shared memory (or unused when args.bias == nullptr).
// [c_begin, c_end): the tile columns this thread writes (multiples of 16; default all BN).
__device__ __forceinline__ void epi_store_strided(const TcArgs& args, uint32_t taddr, bool row_ok, long long rbase,
                                                  int col0, int cbase, const float* bs, int c_begin = 0,
                                                  int c_end = 1 << 30) {
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
        if (args.relu_top) {   // ReLU backward folded in: keep where the ReLU output is positive
#pragma unroll
            for (int j = 0; j < 16; j++) {
                if (j < nvalid) {
                    const float r = args.relu_top_bf16
                                        ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(args.relu_top)[off0 + j * args.s_c])
                                        : reinterpret_cast<const float*>(args.relu_top)[off0 + j * args.s_c];
                    x[j] = r > 0.f ? x[j] : 0.f;
                }
            }
        }
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
    // two 16-column TMEM loads in flight per wait (measured: batching four per wait was slower --
    // conv1 forward 96 -> 120 us)
    const int cend = min(args.BN, c_end);
    for (int c0 = c_begin; c0 < cend; c0 += 32) {
        if (col0 + c0 >= args.N) break;  // warp-uniform
        const bool two = c0 + 16 < cend && col0 + c0 + 16 < args.N;
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
        if (args.relu_top) {   // ReLU backward folded in (channels-last BF16 reference, row m = row0 + lane)
            const int m = row0 + lane;
            if (m < args.M) {
                const int img = m / args.P, pix = m - img * args.P;
                const uint4* r4 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(args.relu_top) +
                                                                 (long long)img * args.s_n + (long long)pix * args.s_p +
                                                                 ccol + c0);
                // (host: BF16 output and reference, N a multiple of 64 -- whole 64-column chunks)
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const uint4 rv = r4[j];
                    const uint32_t w4[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        const uint16_t h = (uint16_t)(w4[e >> 1] >> ((e & 1) * 16));
                        const bool pos = (h & 0x8000u) == 0 && (h & 0x7fffu) != 0;   // > 0 (no NaN inputs)
                        x[8 * j + e] = pos ? x[8 * j + e] : 0.f;
                    }
                }
            }
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

// Fused SGD form (inner-product weight gradient, caffe_ip_backward_weight_sgd): the accumulator
// is dW for this warp's 32 weight rows; each lane reads its row's W and momentum (32 FP32 columns,
// full 128-byte lines), applies sgd1 (the update kernel's arithmetic, bit for bit), and stages W, v
// (128-byte swizzle) and the BF16 copy (64-byte swizzle) for three tensor stores -- dW itself never
// reaches memory.  Two 10 KB buffers per warp keep one store group in flight.  Host guarantees:
// beta 0, N a multiple of 32, FP32 W/v rows 16-byte aligned.
__device__ __forceinline__ void epi_sgd_tma(const TcArgs& args, const CUtensorMap* mapW, const CUtensorMap* mapV,
                                            const CUtensorMap* mapWb, uint32_t taddr, int row0, int col0, int ccol,
                                            uint8_t* stage, int& buf, int lane) {
    const int m = row0 + lane;
    const bool row_ok = m < args.M;
    const float* wrow = reinterpret_cast<const float*>(args.out) + (long long)(row_ok ? m : 0) * args.s_n + ccol;
    const float* vrow = args.sgd_v + (long long)(row_ok ? m : 0) * args.s_n + ccol;
    const float lr = args.sgd_lr, mom = args.sgd_mom, decay = args.sgd_decay, gs = args.sgd_gs;
    for (int c0 = 0; c0 < args.BN; c0 += 32) {
        if (col0 + c0 >= args.N) break;   // warp-uniform
        uint32_t g[32];
        tmem_ld16(taddr + c0, *reinterpret_cast<uint32_t(*)[16]>(&g[0]));
        tmem_ld16(taddr + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&g[16]));
        float w[32], v[32];
        {
            const float4* w4 = reinterpret_cast<const float4*>(wrow + c0);
            const float4* v4 = reinterpret_cast<const float4*>(vrow + c0);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const float4 a = w4[q], b = v4[q];
                w[4 * q] = a.x; w[4 * q + 1] = a.y; w[4 * q + 2] = a.z; w[4 * q + 3] = a.w;
                v[4 * q] = b.x; v[4 * q + 1] = b.y; v[4 * q + 2] = b.z; v[4 * q + 3] = b.w;
            }
        }
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; j++) sgd1(w[j], __uint_as_float(g[j]), v[j], lr, mom, decay, gs);
        if (lane == 0) tma_store_wait_read1();
        __syncwarp();
        uint8_t* st = stage + buf * 10240;
        const int sw = lane & 7, sw64 = (lane >> 1) & 3;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            *reinterpret_cast<float4*>(st + lane * 128 + ((j ^ sw) << 4)) =
                make_float4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            *reinterpret_cast<float4*>(st + 4096 + lane * 128 + ((j ^ sw) << 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
            uint4 pk;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(w[8 * j + 2 * e], w[8 * j + 2 * e + 1]);
            *reinterpret_cast<uint4*>(st + 8192 + lane * 64 + ((j ^ sw64) << 4)) = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_2d(mapW, st, ccol + c0, row0);
            tma_store_2d(mapV, st + 4096, ccol + c0, row0);
            tma_store_2d(mapWb, st + 8192, ccol + c0, row0);
            tma_store_commit();
        }
        buf ^= 1;
    }
}

// Row-staged form for channels-last BF16 outputs (s_c == 1, beta == 0, BN*2 <= 256 bytes): each
// warp stages its 32 rows x BN columns -- a whole row segment per lane, pitch padded to an odd
// number of 16-byte chunks so the staging writes are bank-conflict-free -- then writes the 32
// segments back in memory order, consecutive lanes on consecutive 16-byte pieces.  When a tile's
// columns are all of a pixel's channels (the first conv layer: 96 channels, 192-byte pixels),
// consecutive output pixels are contiguous and every store instruction writes 512 contiguous
// bytes instead of 32 scattered 16-byte pieces.  Bias and ReLU are applied before staging; the
// bytes written are identical to epi_store_strided's.  stage: >= 32 x 17 x 16 bytes.
__device__ __forceinline__ void epi_store_rows(const TcArgs& args, uint32_t taddr, bool row_ok, long long rbase,
                                               int col0, int cbase, const float* bs, uint8_t* stage, int lane) {
    const int nch = args.BN / 8;                // 16-byte pieces per row segment (BN bf16 columns)
    const int pitch = (nch | 1) * 16;           // odd number of chunks per staged row
    const unsigned okmask = __ballot_sync(0xffffffffu, row_ok);
    const int rb_lo = (int)(rbase & 0xffffffffLL), rb_hi = (int)(rbase >> 32);
    uint8_t* st = stage + lane * pitch;
    for (int c0 = 0; c0 < args.BN; c0 += 32) {   // TMEM -> bias/ReLU -> bf16 -> staging, 32 columns at a time
        uint32_t v[32];
        tmem_ld16(taddr + c0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        if (c0 + 16 < args.BN) tmem_ld16(taddr + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        tmem_wait_ld();
        float x[32];
#pragma unroll
        for (int j = 0; j < 32; j++) x[j] = __uint_as_float(v[j]);
        if (args.bias) {
#pragma unroll
            for (int j = 0; j < 32; j++) x[j] += bs[c0 + j];
        }
        if (args.relu) {
#pragma unroll
            for (int j = 0; j < 32; j++) x[j] = x[j] > 0.f ? x[j] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            if (c0 + 8 * q < args.BN) {
                uint4 pk;
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
                for (int e = 0; e < 4; e++) h2[e] = __floats2bfloat162_rn(x[8 * q + 2 * e], x[8 * q + 2 * e + 1]);
                *reinterpret_cast<uint4*>(st + (c0 / 8 + q) * 16) = pk;
            }
        }
    }
    __syncwarp();
    if (okmask != 0) {
        const int nvalid = min(args.BN, args.N - col0);     // valid columns of the tile
        const unsigned inv = (65536u + nch - 1) / nch;      // q / nch for q < 512
        for (int it = 0; it < nch; it++) {
            const int q = it * 32 + lane;
            const int row = (int)(((unsigned)q * inv) >> 16), j = q - row * nch;
            const long long rb = (long long)(unsigned)__shfl_sync(0xffffffffu, rb_lo, row) |
                                 ((long long)__shfl_sync(0xffffffffu, rb_hi, row) << 32);
            if (((okmask >> row) & 1u) && j * 8 < nvalid) {
                const uint4 val = *reinterpret_cast<const uint4*>(stage + row * pitch + j * 16);
                *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(args.out) + rb + cbase + j * 8) = val;
            }
        }
    }
    __syncwarp();
}

}  // namespace cb
