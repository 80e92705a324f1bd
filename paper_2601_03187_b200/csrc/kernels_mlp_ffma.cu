// N7: the fp32 CUDA-core reference chain of TaNG's residual MLP (the "1e-5 fp32 path"):
// fp32 weights and activations, fp32 arithmetic throughout -- every product and sum is an fp32
// FFMA/FADD, accumulated with error-free transformations (TwoProduct via FMA, TwoSum) so the
// dot products are as accurate as a twice-longer mantissa; the only rounding left is the fp32
// store of each activation (R7).
//
// P:371 (§6.1): an initial FC layer S->N, B residual blocks, a final FC N->C; ReLU throughout.
// Eq. (1) P:377 (balanced reading):  B(x) = A(A(x.w1 + b1).w2 + b2 + x).
// the predicted tuple is the argmax of the outputs (ties -> lowest index).
// Features are fused: each packet's 7 segments are formed in registers from its header.
//
// A block owns 32 packets; activations live in shared memory as fp32 [32][N]; weights are
// streamed from L2 ([in][out], coalesced across the 128 output columns a warp-pair covers).
// This path is a correctness reference, not the throughput path (that is kernels_mlp_tc.cu).
#include <cfloat>

#include "tang_internal.h"

namespace tang {
namespace {

constexpr int kRows = 32;
constexpr int kThreads = 256;
constexpr int kColChunk = 128;        // output columns per pass; 2 row groups x 16 rows
constexpr uint32_t kFull = 0xFFFFFFFFu;

// out[r][c] = act( sum_k in[r][k] W[k][c] + b[c] (+ skip[r][c]) ), for all 32 rows, c < ncol
template <bool kRelu, bool kSkip>
__device__ void layer(const float* __restrict__ in, int K, const float* __restrict__ W, const float* __restrict__ b,
                      int ncol, float* out, int ld_in, int ld_out) {
    const int j = threadIdx.x & (kColChunk - 1);
    const int g = threadIdx.x >> 7;     // 0..1
    for (int c0 = 0; c0 < ncol; c0 += kColChunk) {
        const int c = c0 + j;
        // compensated fp32 dot products: s + e carries the sum to ~2^-48 relative, so the only
        // rounding that reaches the logits is the fp32 store of each activation (1e-5 at N = 512)
        float sum[16], err[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) { sum[i] = 0.f; err[i] = 0.f; }
        if (c < ncol) {
            for (int k = 0; k < K; ++k) {
                const float w = __ldg(W + size_t(k) * ncol + c);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float a = in[(g + 2 * i) * ld_in + k];
                    // _rn intrinsics: never contracted into FMAs, so the transformations stay exact
                    const float pr = __fmul_rn(a, w);
                    const float pe = __fmaf_rn(a, w, -pr);          // TwoProduct: a*w = pr + pe exactly
                    const float t = __fadd_rn(sum[i], pr);          // TwoSum: sum + pr = t + se exactly
                    const float z = __fsub_rn(t, sum[i]);
                    const float se = __fadd_rn(__fsub_rn(sum[i], __fsub_rn(t, z)), __fsub_rn(pr, z));
                    sum[i] = t;
                    err[i] = __fadd_rn(err[i], __fadd_rn(se, pe));
                }
            }
        }
        __syncthreads();   // every thread done reading `in` columns before anyone writes `out`
        if (c < ncol) {
            const float bc = __ldg(b + c);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int r = g + 2 * i;
                // (sum + err) + b (+ skip) with one more TwoSum, then a single rounding
                float hi = sum[i], lo = err[i];
                auto add = [&](float v) {
                    const float t = __fadd_rn(hi, v), z = __fsub_rn(t, hi);
                    lo = __fadd_rn(lo, __fadd_rn(__fsub_rn(hi, __fsub_rn(t, z)), __fsub_rn(v, z)));
                    hi = t;
                };
                add(bc);
                if (kSkip) add(out[r * ld_out + c]);            // the skip input x lives in `out` (in place)
                float v = __fadd_rn(hi, lo);
                if (kRelu) v = v > 0.f ? v : 0.f;
                out[r * ld_out + c] = v;
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) mlp_ffma_kernel(WeightsF32 w, const void* __restrict__ hdr, size_t n,
                                                            uint32_t k, uint32_t* __restrict__ pred,
                                                            float* __restrict__ logits) {
    extern __shared__ __align__(16) float smem[];
    const int N = w.N, C = w.C;
    const int ldx = N, ldl = (C > N ? C : N);
    float* X = smem;                    // [32][N]  block input / output (in place)
    float* U = smem + kRows * ldx;      // [32][max(N, C)]  inner activation, then logits
    float* F = U + kRows * ldl;         // [32][8]  features
    const size_t row0 = size_t(blockIdx.x) * kRows;

    // a2: encode, one thread per packet
    if (threadIdx.x < kRows) {
        const size_t i = row0 + threadIdx.x;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (i < n) v = __ldg(reinterpret_cast<const uint4*>(hdr) + i);
        const float sc = 1.0f / 65536.0f;
        float* f = F + threadIdx.x * 8;
        f[0] = float(v.x >> 16) * sc;
        f[1] = float(v.x & 0xFFFFu) * sc;
        f[2] = float(v.y >> 16) * sc;
        f[3] = float(v.y & 0xFFFFu) * sc;
        f[4] = float(v.z & 0xFFFFu) * sc;
        f[5] = float(v.z >> 16) * sc;
        f[6] = float(v.w & 0xFFu) * sc;
        f[7] = 0.f;
    }
    __syncthreads();
    // a3: input FC + ReLU
    layer<true, false>(F, kS, w.W0, w.b0, N, X, 8, ldx);
    // a4: residual blocks
    for (int b = 0; b < w.B; ++b) {
        const size_t off = size_t(b) * N * N;
        layer<true, false>(X, N, w.W1 + off, w.b1 + size_t(b) * N, N, U, ldx, ldl);
        layer<true, true>(U, N, w.W2 + off, w.b2 + size_t(b) * N, N, X, ldl, ldx);
    }
    // a5: output FC (raw logits, reading 2)
    layer<false, false>(X, N, w.Wo, w.bo, C, U, ldx, ldl);

    // argmax / top-k: one warp per row, ties to the lowest index
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = warp; r < kRows; r += kThreads / 32) {
        const size_t i = row0 + r;
        if (i >= n) continue;
        const float* L = U + r * ldl;
        if (logits) for (int c = lane; c < C; c += 32) logits[i * C + c] = L[c];
        int taken[4];
        for (uint32_t q = 0; q < k; ++q) {
            float bv = -FLT_MAX;
            int bc = 0x7FFFFFFF;
            for (int c = lane; c < C; c += 32) {
                bool used = false;
                for (uint32_t p = 0; p < q; ++p) used |= (taken[p] == c);
                const float v = L[c];
                if (!used && (v > bv || (v == bv && c < bc))) { bv = v; bc = c; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(kFull, bv, o);
                const int oc = __shfl_xor_sync(kFull, bc, o);
                if (ov > bv || (ov == bv && oc < bc)) { bv = ov; bc = oc; }
            }
            taken[q] = bc;
            if (lane == 0) pred[i * k + q] = uint32_t(bc);
        }
    }
}

}  // namespace

void launch_mlp_ffma(const WeightsF32& w, const void* hdr, size_t n, uint32_t k, uint32_t* pred, float* logits,
                     cudaStream_t s) {
    if (n == 0) return;
    const int ldl = w.C > w.N ? w.C : w.N;
    const size_t smem = sizeof(float) * (size_t(kRows) * w.N + size_t(kRows) * ldl + kRows * 8);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(mlp_ffma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_set = true;
    }
    mlp_ffma_kernel<<<unsigned((n + kRows - 1) / kRows), kThreads, smem, s>>>(w, hdr, n, k, pred, logits);
}

}  // namespace tang
