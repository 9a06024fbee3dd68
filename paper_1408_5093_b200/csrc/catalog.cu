// catalog.cu -- the rest of the paper's layer catalogue (Sec. 3.2: "nonlinearities like
// rectified linear and logistic ... element-wise operations ... losses like softmax and hinge") and
// the device side of the solver (Sec. 3.4: "learning rate decay schedules, momentum").
//
//   sigmoid          S:199 / S:208  (backward from the forward output, in-place allowed)
//   eltwise          S:235 / S:244  sum (coefficients), product, max (first input wins ties)
//   hinge loss       S:271          one-vs-all L1 hinge, deterministic fixed-order mean
//   solver           S:514 lr_at_iter (fixed / step / inv), S:523 update with the device-resident
//                    learning rate, S:524 divergence guard (a non-finite loss freezes the parameters)
//
// All elementwise kernels are HBM-bound streaming kernels: 16-byte vector loads/stores of 8 BF16 or
// 2x4 FP32 values per thread, a grid-stride loop over whole vectors sized to the SM count, and a
// scalar tail.  Elementwise ops are layout-agnostic (every operand has the same layout).
#include "internal.h"
#include "ptx.cuh"
#include <algorithm>
#include <cmath>

#include <cuda_bf16.h>

namespace cb {

namespace {

inline unsigned grid_for(long long vec, int threads) {
    long long b = (vec + threads - 1) / threads;
    const long long cap = (long long)num_sms() * 8;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

// 8 consecutive elements of an F32 or BF16 buffer as floats
__device__ __forceinline__ void ld8(const void* p, long long v, int bf16, float (&o)[8]) {
    if (bf16) {
        const uint4 u = reinterpret_cast<const uint4*>(p)[v];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const float2 f = __bfloat1622float2(h[e]);
            o[2 * e] = f.x;
            o[2 * e + 1] = f.y;
        }
    } else {
        const float4 a = reinterpret_cast<const float4*>(p)[2 * v];
        const float4 b = reinterpret_cast<const float4*>(p)[2 * v + 1];
        o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
        o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
    }
}
__device__ __forceinline__ void st8(void* p, long long v, int bf16, const float (&o)[8]) {
    if (bf16) {
        uint4 u;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; e++) h[e] = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
        reinterpret_cast<uint4*>(p)[v] = u;
    } else {
        reinterpret_cast<float4*>(p)[2 * v] = make_float4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<float4*>(p)[2 * v + 1] = make_float4(o[4], o[5], o[6], o[7]);
    }
}
__device__ __forceinline__ float ld1(const void* p, long long i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]) : reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void st1(void* p, long long i, int bf16, float v) {
    if (bf16) reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(p)[i] = v;
}

// ---------------------------------------------------------------- sigmoid
__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + expf(-x)); }

__global__ void sigmoid_fwd_kernel(const void* __restrict__ x, void* y, int bf16, long long n) {
    const long long nv = n / 8, stride = (long long)gridDim.x * blockDim.x;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv; v += stride) {
        float a[8];
        ld8(x, v, bf16, a);
#pragma unroll
        for (int e = 0; e < 8; e++) a[e] = sigm(a[e]);
        st8(y, v, bf16, a);
    }
    for (long long i = nv * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
        st1(y, i, bf16, sigm(ld1(x, i, bf16)));
}

__global__ void sigmoid_bwd_kernel(const void* __restrict__ y, const void* dy, void* dx, int ybf, int dbf, long long n) {
    const long long nv = n / 8, stride = (long long)gridDim.x * blockDim.x;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv; v += stride) {
        float a[8], g[8];
        ld8(y, v, ybf, a);
        ld8(dy, v, dbf, g);
#pragma unroll
        for (int e = 0; e < 8; e++) g[e] = g[e] * a[e] * (1.f - a[e]);
        st8(dx, v, dbf, g);
    }
    for (long long i = nv * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float a = ld1(y, i, ybf);
        st1(dx, i, dbf, ld1(dy, i, dbf) * a * (1.f - a));
    }
}

// ---------------------------------------------------------------- eltwise
struct EltArgs {
    const void* in[ELT_MAX_INPUTS];
    void* out[ELT_MAX_INPUTS];          // backward: one diff per input
    float coeff[ELT_MAX_INPUTS];
    int n_in, op, bf16;
};

template <int OP>
__device__ __forceinline__ float elt_combine(const float (&x)[ELT_MAX_INPUTS], const EltArgs& a) {
    float acc = OP == ELT_SUM ? a.coeff[0] * x[0] : x[0];
#pragma unroll
    for (int i = 1; i < ELT_MAX_INPUTS; i++) {
        if (i < a.n_in) {
            if (OP == ELT_SUM) acc = fmaf(a.coeff[i], x[i], acc);
            else if (OP == ELT_PROD) acc *= x[i];
            else acc = x[i] > acc ? x[i] : acc;   // strict: the first input wins ties
        }
    }
    return acc;
}

template <int OP>
__global__ void eltwise_fwd_kernel(const EltArgs a, void* __restrict__ y, long long n) {
    const long long nv = n / 8, stride = (long long)gridDim.x * blockDim.x;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv; v += stride) {
        float xs[ELT_MAX_INPUTS][8];
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++)
            if (i < a.n_in) ld8(a.in[i], v, a.bf16, xs[i]);
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            float x[ELT_MAX_INPUTS];
#pragma unroll
            for (int i = 0; i < ELT_MAX_INPUTS; i++) x[i] = i < a.n_in ? xs[i][e] : 0.f;
            o[e] = elt_combine<OP>(x, a);
        }
        st8(y, v, a.bf16, o);
    }
    for (long long q = nv * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += stride) {
        float x[ELT_MAX_INPUTS];
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++) x[i] = i < a.n_in ? ld1(a.in[i], q, a.bf16) : 0.f;
        st1(y, q, a.bf16, elt_combine<OP>(x, a));
    }
}

// diff_i of one element: sum -> coeff_i * dy; prod -> dy * prod_{j != i} x_j (ascending j, no
// division by x_i); max -> dy at the first input holding the maximum, 0 elsewhere
template <int OP>
__device__ __forceinline__ void elt_diffs(const float (&x)[ELT_MAX_INPUTS], float g, const EltArgs& a,
                                          float (&d)[ELT_MAX_INPUTS]) {
    if (OP == ELT_SUM) {
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++) d[i] = a.coeff[i] * g;
    } else if (OP == ELT_PROD) {
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++) {
            float p = 1.f;
#pragma unroll
            for (int j = 0; j < ELT_MAX_INPUTS; j++)
                if (j != i && j < a.n_in) p *= x[j];
            d[i] = g * p;
        }
    } else {
        int arg = 0;
        float best = x[0];
#pragma unroll
        for (int i = 1; i < ELT_MAX_INPUTS; i++)
            if (i < a.n_in && x[i] > best) { best = x[i]; arg = i; }
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++) d[i] = i == arg ? g : 0.f;
    }
}

template <int OP>
__global__ void eltwise_bwd_kernel(const EltArgs a, const void* __restrict__ dy, long long n) {
    const long long nv = n / 8, stride = (long long)gridDim.x * blockDim.x;
    constexpr bool need_x = OP != ELT_SUM;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv; v += stride) {
        float xs[ELT_MAX_INPUTS][8], g[8];
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++)
            if (need_x && i < a.n_in) ld8(a.in[i], v, a.bf16, xs[i]);
        ld8(dy, v, a.bf16, g);
        float ds[ELT_MAX_INPUTS][8];
#pragma unroll
        for (int e = 0; e < 8; e++) {
            float x[ELT_MAX_INPUTS], d[ELT_MAX_INPUTS];
#pragma unroll
            for (int i = 0; i < ELT_MAX_INPUTS; i++) x[i] = (need_x && i < a.n_in) ? xs[i][e] : 0.f;
            elt_diffs<OP>(x, g[e], a, d);
#pragma unroll
            for (int i = 0; i < ELT_MAX_INPUTS; i++) ds[i][e] = d[i];
        }
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++)
            if (i < a.n_in) st8(a.out[i], v, a.bf16, ds[i]);
    }
    for (long long q = nv * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += stride) {
        float x[ELT_MAX_INPUTS], d[ELT_MAX_INPUTS];
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++) x[i] = (need_x && i < a.n_in) ? ld1(a.in[i], q, a.bf16) : 0.f;
        elt_diffs<OP>(x, ld1(dy, q, a.bf16), a, d);
#pragma unroll
        for (int i = 0; i < ELT_MAX_INPUTS; i++)
            if (i < a.n_in) st1(a.out[i], q, a.bf16, d[i]);
    }
}

// ---------------------------------------------------------------- hinge loss
// One block of 32 warps, warp w owns rows w, w+32, ...; a lane sums its columns in ascending order,
// the warp reduces with a fixed butterfly, then thread 0 adds the warps in order: deterministic.
// A label outside [0, K) is never used as an index; its row's loss term and diff are NaN.
__global__ void __launch_bounds__(1024, 1)
hinge_loss_kernel(const void* __restrict__ s, int sbf, const int32_t* __restrict__ labels, float* __restrict__ loss,
                  void* __restrict__ diff, int dbf, int N, int K) {
    __shared__ float wsum[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float invN = 1.f / N;
    float my = 0.f;
    for (int n = warp; n < N; n += 32) {
        const int lab = labels[n];
        const bool ok = (unsigned)lab < (unsigned)K;
        const float bad = ok ? 0.f : __int_as_float(0x7fc00000);
        const long long base = (long long)n * K;
        float rs = 0.f;
        for (int k = lane; k < K; k += 32) {
            const float y = k == lab ? 1.f : -1.f;
            const float m = 1.f - y * ld1(s, base + k, sbf);
            if (m > 0.f) rs += m;
            if (diff) st1(diff, base + k, dbf, (m > 0.f ? -y * invN : 0.f) + bad);
        }
        for (int o = 16; o; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
        my += rs + bad;
    }
    if (lane == 0) wsum[warp] = my;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < 32; w++) t += wsum[w];
        *loss = t * invN;
    }
}

// ---------------------------------------------------------------- solver (device state)
__device__ double lr_policy_eval(const LrPolicy& p, long long it) {
    if (p.policy == LR_STEP) return (double)p.base_lr * pow((double)p.gamma, (double)(it / p.stepsize));
    if (p.policy == LR_INV) return (double)p.base_lr * pow(1.0 + (double)p.gamma * (double)it, -(double)p.power);
    return (double)p.base_lr;
}

__global__ void solver_begin_kernel(const LrPolicy p, SolverDev* st, const float* loss) {
    SolverDev s = *st;
    if (loss && !isfinite(*loss) && !s.diverged) {
        s.diverged = 1;
        s.diverged_iter = s.iter;
    }
    s.lr = (float)lr_policy_eval(p, s.iter);
    if (loss) s.last_loss = *loss;
    *st = s;
}

__global__ void solver_end_kernel(SolverDev* st) {
    if (!st->diverged) st->iter += 1;
}

// The update kernel of simple.cu with the learning rate read from the solver state; a diverged
// state (non-finite loss seen) leaves w, v and the BF16 copy untouched.
__global__ void __launch_bounds__(256, 5)
sgd_solver_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ v,
                  __nv_bfloat16* __restrict__ wb, long long n, const SolverDev* __restrict__ st, float mom, float decay,
                  float gs) {
    if (st->diverged) return;
    const float lr = st->lr;
    const long long n4 = n / 4;
    const long long stride = (long long)gridDim.x * blockDim.x;
    float4* w4 = reinterpret_cast<float4*>(w);
    float4* v4 = reinterpret_cast<float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n4; t += stride) {
        float4 wa = w4[t], va = v4[t];
        const float4 ga = g4[t];
        sgd1(wa.x, ga.x, va.x, lr, mom, decay, gs);
        sgd1(wa.y, ga.y, va.y, lr, mom, decay, gs);
        sgd1(wa.z, ga.z, va.z, lr, mom, decay, gs);
        sgd1(wa.w, ga.w, va.w, lr, mom, decay, gs);
        v4[t] = va;
        w4[t] = wa;
        if (wb) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(wa.x, wa.y), hi = __floats2bfloat162_rn(wa.z, wa.w);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&lo);
            pk.y = *reinterpret_cast<uint32_t*>(&hi);
            reinterpret_cast<uint2*>(wb)[t] = pk;
        }
    }
    for (long long q = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += stride) {
        float nw = w[q], vv = v[q];
        sgd1(nw, g[q], vv, lr, mom, decay, gs);
        v[q] = vv;
        w[q] = nw;
        if (wb) wb[q] = __float2bfloat16_rn(nw);
    }
}

}  // namespace

cudaError_t sigmoid_fwd_k(const void* x, void* y, int bf16, long long n, cudaStream_t s) {
    sigmoid_fwd_kernel<<<grid_for(n / 8 + 1, 256), 256, 0, s>>>(x, y, bf16, n);
    note_launch();
    return cudaGetLastError();
}

cudaError_t sigmoid_bwd_k(const void* y, const void* dy, void* dx, int y_bf16, int d_bf16, long long n, cudaStream_t s) {
    sigmoid_bwd_kernel<<<grid_for(n / 8 + 1, 256), 256, 0, s>>>(y, dy, dx, y_bf16, d_bf16, n);
    note_launch();
    return cudaGetLastError();
}

cudaError_t eltwise_fwd_k(int op, int n_in, const void* const* in, const float* coeff, void* y, int bf16, long long n,
                          cudaStream_t s) {
    EltArgs a = {};
    a.n_in = n_in;
    a.op = op;
    a.bf16 = bf16;
    for (int i = 0; i < n_in; i++) {
        a.in[i] = in[i];
        a.coeff[i] = coeff ? coeff[i] : 1.f;
    }
    const unsigned grid = grid_for(n / 8 + 1, 256);
    if (op == ELT_SUM) eltwise_fwd_kernel<ELT_SUM><<<grid, 256, 0, s>>>(a, y, n);
    else if (op == ELT_PROD) eltwise_fwd_kernel<ELT_PROD><<<grid, 256, 0, s>>>(a, y, n);
    else eltwise_fwd_kernel<ELT_MAX><<<grid, 256, 0, s>>>(a, y, n);
    note_launch();
    return cudaGetLastError();
}

cudaError_t eltwise_bwd_k(int op, int n_in, const void* const* in, const float* coeff, const void* dy,
                          void* const* dx, int bf16, long long n, cudaStream_t s) {
    EltArgs a = {};
    a.n_in = n_in;
    a.op = op;
    a.bf16 = bf16;
    for (int i = 0; i < n_in; i++) {
        a.in[i] = in ? in[i] : nullptr;
        a.out[i] = dx[i];
        a.coeff[i] = coeff ? coeff[i] : 1.f;
    }
    const unsigned grid = grid_for(n / 8 + 1, 256);
    if (op == ELT_SUM) eltwise_bwd_kernel<ELT_SUM><<<grid, 256, 0, s>>>(a, dy, n);
    else if (op == ELT_PROD) eltwise_bwd_kernel<ELT_PROD><<<grid, 256, 0, s>>>(a, dy, n);
    else eltwise_bwd_kernel<ELT_MAX><<<grid, 256, 0, s>>>(a, dy, n);
    note_launch();
    return cudaGetLastError();
}

cudaError_t hinge_loss_k(const void* scores, int bf16, const int32_t* labels, float* loss, void* diff, int diff_bf16,
                         int N, int K, cudaStream_t s) {
    hinge_loss_kernel<<<1, 1024, 0, s>>>(scores, bf16, labels, loss, diff, diff_bf16, N, K);
    note_launch();
    return cudaGetLastError();
}

double lr_policy_host(const LrPolicy& p, long long it) {
    if (p.policy == LR_STEP) return (double)p.base_lr * std::pow((double)p.gamma, (double)(it / p.stepsize));
    if (p.policy == LR_INV) return (double)p.base_lr * std::pow(1.0 + (double)p.gamma * (double)it, -(double)p.power);
    return (double)p.base_lr;
}

cudaError_t solver_begin_k(const LrPolicy& p, SolverDev* st, const float* loss, cudaStream_t s) {
    solver_begin_kernel<<<1, 1, 0, s>>>(p, st, loss);
    note_launch();
    return cudaGetLastError();
}

cudaError_t solver_end_k(SolverDev* st, cudaStream_t s) {
    solver_end_kernel<<<1, 1, 0, s>>>(st);
    note_launch();
    return cudaGetLastError();
}

cudaError_t sgd_solver_k(float* w, const float* g, float* v, void* w_bf16, long long count, const SolverDev* st,
                         float mom, float decay, float gscale, cudaStream_t s) {
    static bool carve = false;
    if (!carve) {
        cudaFuncSetAttribute(sgd_solver_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        carve = true;
    }
    const int threads = g_sgd_threads;
    const long long want = (count / 4 + threads - 1) / threads;
    const int grid = (int)std::max(1LL, std::min<long long>((long long)num_sms() * g_sgd_blocks_per_sm, want));
    sgd_solver_kernel<<<grid, threads, 0, s>>>(w, g, v, (__nv_bfloat16*)w_bf16, count, st, mom, decay, gscale);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cb
