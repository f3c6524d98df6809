// Top-1 router on the device (the step on the near side of
// the path). Restates RouterSim.assign (reference pipeline.py:164-182):
//
//  ARGMAX  scores[t][e] = sum_k f64(x[t][k]) * proj[k][e] (+ bias[e]), in
//          float64 as the reference; id = argmax over e, the lowest index on
//          ties (np.argmax); gate[t] = softmax(scores[t])[id] (float32) for
//          combine scaling — the reference has no gate, so it is optional.
//  HASH    h = sum_k u64(bits(f32 x[t][k])) * mult[k]  (u64, wrapping), then
//          h ^= h >> 33; h *= 0xFF51AFD7ED558CCD; h ^= h >> 33; id = h % E.
//          Wrapping u64 sums are order-free, so this is bit-exact.
//
// ARGMAX runs as two launches: a score kernel (a CTA = 32 experts, one per
// lane, x R_TOK tokens x one slice of the reduction over k, slices chosen so
// small steps still cover the SMs; partials combined in a fixed order, so
// scores are deterministic) and a select kernel (one CTA per token: slice
// sum, arg-max, softmax). Router matrices are d x E f64 (0.8 MB for
// Switch-base-128, 34 MB for c2048) and read once per step.

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "qmoe.h"
#include "qmoe_internal.h"

namespace {

constexpr int R_WARPS = 8;
constexpr int R_TOK = 8;  // tokens per score CTA (each proj load feeds R_TOK FMAs)

__device__ __forceinline__ double load_xd(const void* x, int bf16, int64_t i) {
  if (bf16) {
    const unsigned short b = reinterpret_cast<const unsigned short*>(x)[i];
    return (double)__uint_as_float(uint32_t(b) << 16);
  }
  return (double)reinterpret_cast<const float*>(x)[i];
}

__device__ __forceinline__ uint32_t load_xbits(const void* x, int bf16, int64_t i) {
  if (bf16) return uint32_t(reinterpret_cast<const unsigned short*>(x)[i]) << 16;
  return __float_as_uint(reinterpret_cast<const float*>(x)[i]);
}

struct ScoreParams {
  const void* x;
  int x_bf16;
  int64_t ldx;
  int T, d, E, ks;
  const double* proj;  // d x E row-major
  double* part;        // ks x T x E partial sums (slice z of the reduction over k)
};

// One CTA = 32 experts (a lane each) x R_TOK tokens x one of ks slices of the
// reduction over k; its 8 warps split the slice again and add their partials
// in a fixed order. Each lane keeps 16 projection loads in flight (the loop
// is load-latency-bound otherwise); x comes from shared memory.
__global__ void __launch_bounds__(R_WARPS * 32) route_score_kernel(ScoreParams P) {
  extern __shared__ __align__(16) float xs[];  // R_TOK x slice tokens of x (f32, exact)
  __shared__ double part[R_WARPS][R_TOK][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int t0 = blockIdx.y * R_TOK;
  const int nt = min(R_TOK, P.T - t0);
  const int z = blockIdx.z;
  const int s0 = (int)((int64_t)P.d * z / P.ks), s1 = (int)((int64_t)P.d * (z + 1) / P.ks);
  const int sl = (s1 - s0 + 3) & ~3;  // row pitch of xs (16-byte rows)
  for (int i = threadIdx.x; i < R_TOK * sl; i += blockDim.x) {
    const int j = i / sl, k = s0 + i % sl;
    xs[i] = (j < nt && k < s1) ? (float)load_xd(P.x, P.x_bf16, (int64_t)(t0 + j) * P.ldx + k) : 0.f;
  }
  __syncthreads();
  // warp w takes k in [k0, k1) of the slice (4-aligned starts: float4 x reads)
  const int q = ((sl >> 2) + R_WARPS - 1) / R_WARPS;
  const int k0 = min(sl, 4 * q * warp), k1 = min(s1 - s0, 4 * q * (warp + 1));
  double acc[R_TOK];
#pragma unroll
  for (int j = 0; j < R_TOK; ++j) acc[j] = 0.0;
  if (e < P.E) {
    const double* pp = P.proj + (int64_t)s0 * P.E + e;
    int k = k0;
    constexpr int KU = 16;  // projection loads in flight per lane
    for (; k + KU <= k1; k += KU) {
      double pk[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) pk[u] = __ldg(pp + (int64_t)(k + u) * P.E);
#pragma unroll
      for (int u4 = 0; u4 < KU; u4 += 4) {
#pragma unroll
        for (int j = 0; j < R_TOK; ++j) {
          const float4 xv = *reinterpret_cast<const float4*>(xs + j * sl + k + u4);
          acc[j] = fma((double)xv.x, pk[u4], acc[j]);
          acc[j] = fma((double)xv.y, pk[u4 + 1], acc[j]);
          acc[j] = fma((double)xv.z, pk[u4 + 2], acc[j]);
          acc[j] = fma((double)xv.w, pk[u4 + 3], acc[j]);
        }
      }
    }
    for (; k < k1; ++k) {
      const double p = __ldg(pp + (int64_t)k * P.E);
#pragma unroll
      for (int j = 0; j < R_TOK; ++j) acc[j] = fma((double)xs[j * sl + k], p, acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < R_TOK; ++j) part[warp][j][lane] = acc[j];
  __syncthreads();
  if (warp == 0 && e < P.E) {
    for (int j = 0; j < nt; ++j) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < R_WARPS; ++w) s += part[w][j][lane];
      P.part[((int64_t)z * P.T + t0 + j) * P.E + e] = s;
    }
  }
}

// One CTA per token: score = sum of the ks partials in slice order + bias
// (written back into slice 0), arg-max with the lowest index on ties, and the
// softmax probability of the winner (block reductions; E up to thousands).
constexpr int SEL_THREADS = 256;

__device__ __forceinline__ void better(double& best, int& bi, double v, int i) {
  if (v > best || (v == best && i < bi)) {
    best = v;
    bi = i;
  }
}

__global__ void __launch_bounds__(SEL_THREADS) route_select_kernel(double* __restrict__ part, int ks, int T, int E,
                                                                   const double* __restrict__ bias, int32_t* assign,
                                                                   float* gate) {
  __shared__ double sv[SEL_THREADS / 32];
  __shared__ int si[SEL_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x;
  double* s = part + (int64_t)t * E;
  double best = -INFINITY;
  int bi = 0x7FFFFFFF;
  for (int e = threadIdx.x; e < E; e += SEL_THREADS) {
    double v = s[e];
    for (int z = 1; z < ks; ++z) v += part[((int64_t)z * T + t) * E + e];
    if (bias) v += bias[e];
    s[e] = v;
    better(best, bi, v, e);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1)
    better(best, bi, __shfl_xor_sync(0xFFFFFFFFu, best, d), __shfl_xor_sync(0xFFFFFFFFu, bi, d));
  if (lane == 0) {
    sv[warp] = best;
    si[warp] = bi;
  }
  __syncthreads();
  best = sv[0];
  bi = si[0];
  for (int w = 1; w < SEL_THREADS / 32; ++w) better(best, bi, sv[w], si[w]);
  if (gate) {
    __syncthreads();  // everyone has read sv / si
    double z = 0.0;
    for (int e = threadIdx.x; e < E; e += SEL_THREADS) z += exp(s[e] - best);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) z += __shfl_xor_sync(0xFFFFFFFFu, z, d);
    if (lane == 0) sv[warp] = z;
    __syncthreads();
    if (threadIdx.x == 0) {
      double zt = 0.0;
      for (int w = 0; w < SEL_THREADS / 32; ++w) zt += sv[w];
      gate[t] = (float)(1.0 / zt);
    }
  }
  if (threadIdx.x == 0) assign[t] = bi == 0x7FFFFFFF ? 0 : bi;
}

__global__ void route_hash_kernel(const void* x, int x_bf16, int64_t ldx, int T, int d, int E,
                                  const uint64_t* __restrict__ mult, int32_t* assign, float* gate) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  uint64_t h = 0;
#pragma unroll 4
  for (int k = lane; k < d; k += 32) h += (uint64_t)load_xbits(x, x_bf16, (int64_t)t * ldx + k) * __ldg(mult + k);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, s);
  if (lane == 0) {
    h ^= h >> 33;
    h *= 0xFF51AFD7ED558CCDull;
    h ^= h >> 33;
    assign[t] = (int32_t)(h % (uint64_t)E);
    if (gate) gate[t] = 1.0f;
  }
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int score_slices(int T, int d, int E) {
  // enough CTAs to cover the SMs about twice; slices of >= 64 k
  const int tiles = ((E + 31) / 32) * ((T + R_TOK - 1) / R_TOK);
  int ks = (2 * 148 + tiles - 1) / tiles;
  ks = std::min(ks, std::max(1, d / 64));
  return std::max(1, std::min(ks, 16));
}

}  // namespace

extern "C" int64_t qmoe_route_scratch(int32_t T, int32_t d, int32_t E) {
  if (T <= 0 || d <= 0 || E <= 0) return 0;
  return (int64_t)score_slices(T, d, E) * T * E;
}

extern "C" int qmoe_route(int rule, const void* d_x, int x_dtype, int64_t ldx, int32_t T, int32_t d, int32_t E,
                          const double* d_proj, const double* d_bias, const uint64_t* d_mult, double* d_scores,
                          int32_t* d_assign, float* d_gate, void* stream) {
  if (!d_x || T < 0 || d <= 0 || E < 1 || ldx < d || !d_assign || (x_dtype != QMOE_X_F32 && x_dtype != QMOE_X_BF16))
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (T == 0) return QMOE_OK;
  const int bf16 = x_dtype == QMOE_X_BF16;
  const int wpb = 8;  // warps per block of the per-token kernels
  if (rule == QMOE_ROUTE_HASH) {
    if (!d_mult) return qmoe::fail(QMOE_EINVAL, "hash rule needs mult");
    route_hash_kernel<<<(T + wpb - 1) / wpb, wpb * 32, 0, S(stream)>>>(d_x, bf16, ldx, T, d, E, d_mult, d_assign,
                                                                      d_gate);
  } else if (rule == QMOE_ROUTE_ARGMAX) {
    if (!d_proj || !d_scores) return qmoe::fail(QMOE_EINVAL, "argmax rule needs proj and a scores buffer");
    const int ks = score_slices(T, d, E);
    ScoreParams P{d_x, bf16, ldx, T, d, E, ks, d_proj, d_scores};
    dim3 grid((E + 31) / 32, (T + R_TOK - 1) / R_TOK, ks);
    const int sl = ((d + ks - 1) / ks + 3 + 3) & ~3;
    const size_t smem = (size_t)R_TOK * sl * sizeof(float);
    if (smem > 48 * 1024) {
      const cudaError_t ae =
          cudaFuncSetAttribute(route_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (ae != cudaSuccess) return qmoe::fail(QMOE_ECUDA, cudaGetErrorString(ae));
    }
    route_score_kernel<<<grid, R_WARPS * 32, smem, S(stream)>>>(P);
    route_select_kernel<<<T, SEL_THREADS, 0, S(stream)>>>(d_scores, ks, T, E, d_bias, d_assign, d_gate);
  } else {
    return qmoe::fail(QMOE_EINVAL, "unknown routing rule");
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return qmoe::fail(QMOE_ECUDA, cudaGetErrorString(e));
  return QMOE_OK;
}
