// Device half of libqmoe (sm_100a): dictionary upload, row validation,
// decompress, fused decode + matvec (grouped/persistent, sparse-table and
// general paths), the paper's Listing-1 kernel with lane trace, the GPU
// encoder, RTN quantizer and the MoE dispatcher planner.
//
// Reference semantics cited per kernel (paths relative to
// /root/reference/pkg/src/moepack/ unless noted).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "qmoe.h"
#include "qmoe_internal.h"

#define FULL_MASK 0xffffffffu

struct qmoe_dict {
  int device = 0;
  uint64_t hash64 = 0;
  int max_nz = 0;
  int sparse_ok = 0;
  int num_sms = 148;
  int max_smem_optin = 0;
  uint32_t* d_words = nullptr;   // (65536, 2) decode words
  uint32_t* d_stab = nullptr;    // sparse entry table (see qmoe_internal.h)
  uint8_t* d_len = nullptr;      // 2n per entry
  int32_t* d_next = nullptr;     // trie next_node (65537, 9)
};

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  return qmoe::fail(QMOE_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr, what)                           \
  do {                                           \
    cudaError_t _e = (expr);                     \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- numerics
// f32_to_bf16_bits + widen (bf16.py:11-30): RNE on the u32 pattern, no NaN case.
__device__ __forceinline__ float bf16_round_dev(float v) {
  uint32_t u = __float_as_uint(v);
  u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
  return __uint_as_float(u);
}
__device__ __forceinline__ float bf16_lo(uint32_t mm) { return __uint_as_float(mm << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t mm) { return __uint_as_float(mm & 0xFFFF0000u); }

__device__ __forceinline__ float load_x(const void* x, int dtype, int64_t i) {
  if (dtype == QMOE_X_BF16) {
    uint16_t b = __ldg(reinterpret_cast<const unsigned short*>(x) + i);
    return __uint_as_float(uint32_t(b) << 16);
  }
  return __ldg(reinterpret_cast<const float*>(x) + i);
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL_MASK, v, d);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL_MASK, v, d);
  return v;
}

__device__ __forceinline__ void flag_bad_row(int32_t* bad, int row) {
  if (bad) {
    atomicAdd(bad, 1);
    atomicMin(bad + 1, row);
  }
}

// ================================================================ validation
// _decode_range row-length check (codec.py:164-169): sum over the row's
// codewords of 2n must equal cols. Warp per row.
__global__ void validate_rows_kernel(const uint8_t* __restrict__ len_tab, const uint16_t* __restrict__ cw,
                                     const int32_t* __restrict__ row_off, int64_t rows, int64_t cols,
                                     int32_t* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    int s = __ldg(row_off + r), e = __ldg(row_off + r + 1);
    int sum = 0;
    for (int i = s + lane; i < e; i += 32) sum += __ldg(len_tab + __ldg(cw + i));
    sum = warp_sum_int(sum);
    if (lane == 0 && (e < s || (int64_t)sum != cols)) flag_bad_row(bad, (int)r);
  }
}

// ================================================================ row walker
// Warp-per-row decode schedule shared by decompress and the fused matvec.
// A row's codewords are split into 32 contiguous lane segments of K = ceil(n/32)
// codewords (one pass covers up to 32*KMAX codewords; longer rows loop).
// Each lane looks its codewords up, sums their lengths, one warp scan gives
// every lane its starting column, then the lane walks its segment.
constexpr int KMAX = 16;

struct SparseTab {
  const uint32_t* smem;      // hot prefix [0, H) staged in shared memory
  int H;
  const uint32_t* __restrict__ gmem;  // full table (cold entries)
  __device__ __forceinline__ uint32_t operator()(uint32_t c) const {
    return c < (uint32_t)H ? smem[c] : __ldg(gmem + c);
  }
};

// ---------------------------------------------------------------- matvec body
// Sparse path: entry -> <= 3 (position, code) slots. Accumulates the two sums
// S1 = sum x over code-1 positions and S2 over code-2 positions per token; the
// row result is bf16_rne(min * S1 + max * S2).
template <int K, int NT>
__device__ __forceinline__ void seg_sparse(const uint16_t* __restrict__ cwp, int cnt, int lane,
                                           const SparseTab& tab, const float* xs, int& base,
                                           float (&a1)[NT], float (&a2)[NT]) {
  const int my0 = lane * K;
  uint32_t t[K];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint32_t e = 0;
    if (my0 + k < cnt) e = tab(__ldg(cwp + my0 + k));
    t[k] = e;
    sum += e & 31u;
  }
  int incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int v = __shfl_up_sync(FULL_MASK, incl, d);
    if (lane >= d) incl += v;
  }
  int off = base + incl - sum;
  base += __shfl_sync(FULL_MASK, incl, 31);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t e = t[k];
    const float* xo = xs + off * NT;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint32_t b = (e >> (8 * j + 8)) & 0xFFu;
      if (b) {
        const float* xp = xo + (b >> 2) * NT;
        float xv[NT];
        if constexpr (NT == 4) {
          float4 v = *reinterpret_cast<const float4*>(xp);
          xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
        } else if constexpr (NT == 2) {
          float2 v = *reinterpret_cast<const float2*>(xp);
          xv[0] = v.x; xv[1] = v.y;
        } else {
#pragma unroll
          for (int q = 0; q < NT; ++q) xv[q] = xp[q];
        }
        if (b & 1u) {
#pragma unroll
          for (int q = 0; q < NT; ++q) a1[q] += xv[q];
        } else {
#pragma unroll
          for (int q = 0; q < NT; ++q) a2[q] += xv[q];
        }
      }
    }
    off += int(e & 31u);
  }
}

// General path (any dictionary, e.g. p0 = 0.7 with up to 6 non-zeros per
// entry): expand the two decode words value by value (dictionary.py:115-120).
template <int K, int NT>
__device__ __forceinline__ void seg_general(const uint16_t* __restrict__ cwp, int cnt, int lane,
                                            const uint32_t* __restrict__ words, const float* xs, int& base,
                                            float (&a1)[NT], float (&a2)[NT]) {
  const int my0 = lane * K;
  uint2 w[K];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    w[k] = make_uint2(0u, 0u);
    if (my0 + k < cnt) w[k] = __ldg(reinterpret_cast<const uint2*>(words) + __ldg(cwp + my0 + k));
    sum += 2 * int(w[k].x & 15u);
  }
  int incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int v = __shfl_up_sync(FULL_MASK, incl, d);
    if (lane >= d) incl += v;
  }
  int off = base + incl - sum;
  base += __shfl_sync(FULL_MASK, incl, 31);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int len = 2 * int(w[k].x & 15u);
    for (int v = 0; v < len; ++v) {
      const uint32_t word = v < 14 ? w[k].x : w[k].y;
      const uint32_t code = (word >> (4 + 2 * (v % 14))) & 3u;
      if (code) {
        const float* xp = xs + (off + v) * NT;
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          if (code == 1u) a1[q] += xp[q];
          else a2[q] += xp[q];
        }
      }
    }
    off += len;
  }
}

template <bool SPARSE, int K, int NT>
__device__ __forceinline__ void seg_dispatch(const uint16_t* cwp, int cnt, int lane, const SparseTab& tab,
                                             const uint32_t* words, const float* xs, int& base,
                                             float (&a1)[NT], float (&a2)[NT]) {
  if constexpr (SPARSE) seg_sparse<K, NT>(cwp, cnt, lane, tab, xs, base, a1, a2);
  else seg_general<K, NT>(cwp, cnt, lane, words, xs, base, a1, a2);
}

template <bool SPARSE, int NT>
__device__ void matvec_row(const qmoe_matrix& m, int r, int lane, const SparseTab& tab,
                           const uint32_t* __restrict__ words, const float* xs, int ntok,
                           const int32_t* tok, float* __restrict__ y, int64_t ldy, int32_t* bad) {
  const int s = __ldg(m.row_off + r), e = __ldg(m.row_off + r + 1);
  const uint32_t mm = __ldg(m.row_minmax + r);
  float a1[NT], a2[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) a1[q] = a2[q] = 0.f;
  int base = 0;
  for (int p = s; p < e; p += 32 * KMAX) {
    const int cnt = min(e - p, 32 * KMAX);
    const int K = (cnt + 31) >> 5;
    const uint16_t* cwp = m.cw + p;
    switch (K) {
#define QMOE_SEG_CASE(KK) \
  case KK: seg_dispatch<SPARSE, KK, NT>(cwp, cnt, lane, tab, words, xs, base, a1, a2); break;
      QMOE_SEG_CASE(1) QMOE_SEG_CASE(2) QMOE_SEG_CASE(3) QMOE_SEG_CASE(4)
      QMOE_SEG_CASE(5) QMOE_SEG_CASE(6) QMOE_SEG_CASE(7) QMOE_SEG_CASE(8)
      QMOE_SEG_CASE(9) QMOE_SEG_CASE(10) QMOE_SEG_CASE(11) QMOE_SEG_CASE(12)
      QMOE_SEG_CASE(13) QMOE_SEG_CASE(14) QMOE_SEG_CASE(15) QMOE_SEG_CASE(16)
#undef QMOE_SEG_CASE
      default: break;
    }
  }
  if (base != m.cols) {  // row decodes to the wrong number of values: never write it
    if (lane == 0) flag_bad_row(bad, r);
    return;
  }
  const float lmin = bf16_lo(mm), lmax = bf16_hi(mm);
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    const float s1 = warp_sum(a1[q]);
    const float s2 = warp_sum(a2[q]);
    if (lane == 0 && q < ntok) {
      float* yp = y + (int64_t)tok[q] * ldy + r;
      *yp = *yp + bf16_round_dev(fmaf(lmin, s1, lmax * s2));
    }
  }
}

// ---------------------------------------------------------------- grouped kernel
struct GroupedParams {
  const uint32_t* stab;
  const uint32_t* words;
  int H;  // hot table entries staged in shared memory
  const qmoe_matrix* mats;
  const qmoe_unit* units;       // nullptr => implicit single-matrix units
  const int32_t* n_units;       // device count (explicit mode)
  int max_units;
  qmoe_matrix single;           // implicit mode
  int rows_per_unit;
  int64_t ntok_single;
  int max_cols;                 // x staging capacity per token
  const void* x;
  int x_dtype;
  int64_t ldx;
  int x_relu;
  float* y;
  int64_t ldy;
  int32_t* bad;
};

__device__ __forceinline__ void get_unit(const GroupedParams& P, int u, qmoe_unit& U, qmoe_matrix& M) {
  if (P.units) {
    U = P.units[u];
    M = P.mats[U.mat];
  } else {
    const int nblk = (P.single.rows + P.rows_per_unit - 1) / P.rows_per_unit;
    const int chunk = u / nblk, blk = u % nblk;
    U.mat = 0;
    U.row0 = blk * P.rows_per_unit;
    U.row1 = min(P.single.rows, U.row0 + P.rows_per_unit);
    const int64_t t0 = (int64_t)chunk * QMOE_NT_MAX;
    U.ntok = (int)(P.ntok_single - t0 < QMOE_NT_MAX ? P.ntok_single - t0 : QMOE_NT_MAX);
#pragma unroll
    for (int q = 0; q < QMOE_NT_MAX; ++q) U.tok[q] = (int)(t0 + min(q, U.ntok - 1));
    M = P.single;
  }
}

template <bool SPARSE, int NT>
__device__ void run_unit(const GroupedParams& P, const qmoe_unit& U, const qmoe_matrix& M,
                         const SparseTab& tab, const float* xs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = U.row0 + warp; r < U.row1; r += nw)
    matvec_row<SPARSE, NT>(M, r, lane, tab, P.words, xs, U.ntok, U.tok, P.y, P.ldy, P.bad);
}

// Persistent grouped decode+matvec: one CTA per SM, the hot prefix of the
// entry table staged in shared memory once per launch, then a contiguous
// slice of work units per CTA (consecutive units usually share x, which then
// stays staged). x is staged as fp32, token-interleaved: xs[col * NT + t].
template <bool SPARSE>
__global__ void __launch_bounds__(512, 1) grouped_matvec_kernel(GroupedParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  uint32_t* tab_s = smem;
  float* xs = reinterpret_cast<float*>(smem + P.H);
  if (SPARSE) {
    const uint4* src = reinterpret_cast<const uint4*>(P.stab);
    uint4* dst = reinterpret_cast<uint4*>(tab_s);
    for (int i = threadIdx.x; i < P.H / 4; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  SparseTab tab{tab_s, SPARSE ? P.H : 0, P.stab};

  int n;
  if (P.units) n = min(*P.n_units, P.max_units);
  else {
    const int nblk = (P.single.rows + P.rows_per_unit - 1) / P.rows_per_unit;
    n = nblk * (int)((P.ntok_single + QMOE_NT_MAX - 1) / QMOE_NT_MAX);
  }
  const int u0 = (int)((int64_t)n * blockIdx.x / gridDim.x);
  const int u1 = (int)((int64_t)n * (blockIdx.x + 1) / gridDim.x);

  int staged_cols = -1, staged_ntok = -1;
  int staged_tok[QMOE_NT_MAX] = {-1, -1, -1, -1};
  for (int u = u0; u < u1; ++u) {
    qmoe_unit U;
    qmoe_matrix M;
    get_unit(P, u, U, M);
    if (U.ntok <= 0 || U.row0 >= U.row1) continue;
    const int nt = U.ntok == 1 ? 1 : (U.ntok == 2 ? 2 : 4);
    bool same = (M.cols == staged_cols) && (nt == staged_ntok);
#pragma unroll
    for (int q = 0; q < QMOE_NT_MAX; ++q) same = same && (q >= U.ntok || U.tok[q] == staged_tok[q]);
    if (!same) {
      __syncthreads();  // every warp is done reading the previous x
      const int ncol = M.cols + 32;  // 32 zero columns absorb padded slots
      for (int i = threadIdx.x; i < ncol * nt; i += blockDim.x) {
        const int c = i / nt, q = i - c * nt;
        float v = 0.f;
        if (c < M.cols && q < U.ntok) {
          v = load_x(P.x, P.x_dtype, (int64_t)U.tok[q] * P.ldx + c);
          if (P.x_relu) v = fmaxf(v, 0.f);
        }
        xs[i] = v;
      }
      staged_cols = M.cols;
      staged_ntok = nt;
#pragma unroll
      for (int q = 0; q < QMOE_NT_MAX; ++q) staged_tok[q] = q < U.ntok ? U.tok[q] : -1;
      __syncthreads();
    }
    if (nt == 1) run_unit<SPARSE, 1>(P, U, M, tab, xs);
    else if (nt == 2) run_unit<SPARSE, 2>(P, U, M, tab, xs);
    else run_unit<SPARSE, 4>(P, U, M, tab, xs);
  }
}

// ================================================================ decompress
// _decode_range (codec.py:158-172) into a zero-initialised (rows, cols) u8
// buffer: only non-zero codes are stored (sparse path) or every value of the
// entry (general path). Same warp-per-row lane-segment schedule.
template <int K>
__device__ __forceinline__ void dseg_sparse(const uint16_t* __restrict__ cwp, int cnt, int lane,
                                            const SparseTab& tab, uint8_t* out, int64_t cols, int& base) {
  const int my0 = lane * K;
  uint32_t t[K];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint32_t e = 0;
    if (my0 + k < cnt) e = tab(__ldg(cwp + my0 + k));
    t[k] = e;
    sum += e & 31u;
  }
  int incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int v = __shfl_up_sync(FULL_MASK, incl, d);
    if (lane >= d) incl += v;
  }
  int off = base + incl - sum;
  base += __shfl_sync(FULL_MASK, incl, 31);
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint32_t b = (t[k] >> (8 * j + 8)) & 0xFFu;
      if (b) {
        const int c = off + int(b >> 2);
        if (c < cols) out[c] = (b & 1u) ? 1 : 2;
      }
    }
    off += int(t[k] & 31u);
  }
}

template <int K>
__device__ __forceinline__ void dseg_general(const uint16_t* __restrict__ cwp, int cnt, int lane,
                                             const uint32_t* __restrict__ words, uint8_t* out, int64_t cols,
                                             int& base) {
  const int my0 = lane * K;
  uint2 w[K];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    w[k] = make_uint2(0u, 0u);
    if (my0 + k < cnt) w[k] = __ldg(reinterpret_cast<const uint2*>(words) + __ldg(cwp + my0 + k));
    sum += 2 * int(w[k].x & 15u);
  }
  int incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int v = __shfl_up_sync(FULL_MASK, incl, d);
    if (lane >= d) incl += v;
  }
  int off = base + incl - sum;
  base += __shfl_sync(FULL_MASK, incl, 31);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int len = 2 * int(w[k].x & 15u);
    for (int v = 0; v < len; ++v) {
      const uint32_t word = v < 14 ? w[k].x : w[k].y;
      const uint32_t code = (word >> (4 + 2 * (v % 14))) & 3u;
      if (code && off + v < cols) out[off + v] = (uint8_t)code;
    }
    off += len;
  }
}

template <bool SPARSE>
__global__ void __launch_bounds__(512) decompress_kernel(const uint32_t* __restrict__ stab,
                                                         const uint32_t* __restrict__ words, int H,
                                                         const uint16_t* __restrict__ cw,
                                                         const int32_t* __restrict__ row_off, int64_t rows,
                                                         int64_t cols, uint8_t* __restrict__ out, int32_t* bad) {
  extern __shared__ __align__(16) uint32_t smem[];
  if (SPARSE) {
    const uint4* src = reinterpret_cast<const uint4*>(stab);
    for (int i = threadIdx.x; i < H / 4; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = __ldg(src + i);
    __syncthreads();
  }
  SparseTab tab{smem, SPARSE ? H : 0, stab};
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += nwarps) {
    const int s = __ldg(row_off + r), e = __ldg(row_off + r + 1);
    uint8_t* orow = out + r * cols;
    int base = 0;
    for (int p = s; p < e; p += 32 * KMAX) {
      const int cnt = min(e - p, 32 * KMAX);
      const int K = (cnt + 31) >> 5;
      switch (K) {
#define QMOE_DSEG(KK)                                                      \
  case KK:                                                                 \
    if (SPARSE) dseg_sparse<KK>(cw + p, cnt, lane, tab, orow, cols, base); \
    else dseg_general<KK>(cw + p, cnt, lane, words, orow, cols, base);     \
    break;
        QMOE_DSEG(1) QMOE_DSEG(2) QMOE_DSEG(3) QMOE_DSEG(4) QMOE_DSEG(5) QMOE_DSEG(6)
        QMOE_DSEG(7) QMOE_DSEG(8) QMOE_DSEG(9) QMOE_DSEG(10) QMOE_DSEG(11) QMOE_DSEG(12)
        QMOE_DSEG(13) QMOE_DSEG(14) QMOE_DSEG(15) QMOE_DSEG(16)
#undef QMOE_DSEG
        default: break;
      }
    }
    if (lane == 0 && base != cols) flag_bad_row(bad, (int)r);
  }
}

// ================================================================ paper kernel
// Listing 1 as written for Ampere, compiled for sm_100a:
// warp per row, x in shared memory as fp32, the dequant table replicated per
// thread to avoid bank conflicts, 32-codeword coalesced block
// fetch, lanes 0..27 extract value (lane % 14) of decode word (lane / 14),
// shuffle reduction. y is fp32 += bf16(res) (reference codec.py:243).
constexpr int PAPER_WARPS = 32;
__global__ void __launch_bounds__(PAPER_WARPS * 32, 1)
    paper_matvec_kernel(const uint32_t* __restrict__ dec, const uint16_t* __restrict__ w_comp,
                        const int32_t* __restrict__ row_off, const uint32_t* __restrict__ minmax,
                        int rows, int cols, const void* x, int x_dtype, float* y, int32_t* trace) {
  extern __shared__ __align__(16) float psm[];
  float* x_shared = psm;                                // cols + 32
  float* deq = psm + cols + 32;                         // [3][32 * warps]
  uint16_t* blk = reinterpret_cast<uint16_t*>(deq + 3 * 32 * PAPER_WARPS);  // [warps][32]
  const int thread = threadIdx.x, lane = thread & 31, warp = thread >> 5;
  for (int i = thread; i < cols + 32; i += blockDim.x) x_shared[i] = i < cols ? load_x(x, x_dtype, i) : 0.f;
  __syncthreads();
  for (int row = blockIdx.x * PAPER_WARPS + warp; row < rows; row += gridDim.x * PAPER_WARPS) {
    const uint32_t mm = __ldg(minmax + row);
    deq[0 * 32 * PAPER_WARPS + thread] = 0.f;
    deq[1 * 32 * PAPER_WARPS + thread] = bf16_lo(mm);
    deq[2 * 32 * PAPER_WARPS + thread] = bf16_hi(mm);
    __syncwarp();
    float res = 0.f;
    int idx = 0;
    const int s = __ldg(row_off + row), n = __ldg(row_off + row + 1) - s;
    for (int i = 0; i < n; i += 32) {
      blk[warp * 32 + lane] = (i + lane < n) ? __ldg(w_comp + s + i + lane) : 0;
      __syncwarp();
      const int m = min(32, n - i);
      for (int j = 0; j < m; ++j) {
        const int enc = blk[warp * 32 + j];
        uint32_t ter = 0, wx14 = 0;
        if (lane < 28) {
          wx14 = __ldg(dec + 2 * enc + lane / 14);
          ter = (wx14 >> (4 + 2 * (lane % 14))) & 3u;
          const float w = deq[ter * 32 * PAPER_WARPS + thread];
          res += w * x_shared[min(idx + lane, cols + 31)];
        }
        if (trace) {  // simulate_warp_row record: {codeword, n, offset, lanes 0-13, lanes 14-27}
          const uint32_t v0 = __reduce_or_sync(FULL_MASK, lane < 14 ? ter << (2 * lane) : 0u);
          const uint32_t v1 = __reduce_or_sync(FULL_MASK, (lane >= 14 && lane < 28) ? ter << (2 * (lane - 14)) : 0u);
          if (lane == 0) {
            int32_t* rec = trace + 5 * (int64_t)(s + i + j);
            rec[0] = enc;
            rec[1] = int(wx14 & 0xF);
            rec[2] = idx;
            rec[3] = (int32_t)v0;
            rec[4] = (int32_t)v1;
          }
        }
        if (lane < 28) idx += 2 * int(wx14 & 0xF);
      }
      __syncwarp();
    }
    res = warp_sum(res);
    if (lane == 0) y[row] = y[row] + bf16_round_dev(res);
    __syncwarp();
  }
}

// ================================================================ encoder
// _encode_rows (codec.py:69-123): per row, follow trie edges; on a stall emit
// the entry of the current node and restart from the root with the same pair
// (every single pair is a root child, dictionary.py:192-193); emit at the end.
// Node i+1 is entry i (dictionary.py:189-190). One thread per row.
template <bool EMIT>
__global__ void encode_kernel(const int32_t* __restrict__ next, const uint8_t* __restrict__ codes, int64_t rows,
                              int64_t cols, int32_t* counts, const int32_t* __restrict__ row_off,
                              uint16_t* __restrict__ cw) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t npair = cols / 2;
  const uint16_t* row = reinterpret_cast<const uint16_t*>(codes + r * cols);
  int node = 0;
  int cnt = 0;
  uint16_t* out = EMIT ? cw + row_off[r] : nullptr;
  for (int64_t i = 0; i < npair; ++i) {
    const uint16_t pr = __ldg(row + i);
    const int sym = 3 * (pr & 0xFF) + (pr >> 8);
    int nx = __ldg(next + node * 9 + sym);
    if (nx < 0) {
      if (EMIT) out[cnt] = (uint16_t)(node - 1);
      ++cnt;
      nx = __ldg(next + sym);
    }
    node = nx;
  }
  if (npair > 0) {
    if (EMIT) out[cnt] = (uint16_t)(node - 1);
    ++cnt;
  }
  if (!EMIT) counts[r] = cnt;
}

__global__ void exclusive_scan_kernel(const int32_t* __restrict__ in, int64_t n, int32_t* out) {
  // single CTA: each thread scans a contiguous chunk, then a block scan of the
  // chunk totals. int64 accumulation; an int32 overflow marks out[n] = -1.
  __shared__ long long part[1024];
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per, e = min(n, b + per);
  long long s = 0;
  for (int64_t i = b; i < e; ++i) s += in[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      long long v = part[i];
      part[i] = acc;
      acc += v;
    }
  }
  __syncthreads();
  long long acc = part[threadIdx.x];
  for (int64_t i = b; i < e; ++i) {
    out[i] = acc > INT32_MAX ? -1 : (int32_t)acc;
    acc += in[i];
  }
  if (e == n && b < e) out[n] = acc > INT32_MAX ? -1 : (int32_t)acc;
  if (n == 0 && threadIdx.x == 0) out[0] = 0;
}

// ================================================================ RTN quantizer
// make_grid (quantize.py:91-107) + rtn_quantize (:219-235) for the ternary
// grid: levels {0, bf16(min), bf16(max)}; nearest level in float64 with ties
// to the smaller magnitude, equal magnitudes in code order (:110-126).
__device__ __forceinline__ uint32_t f32_to_bf16_bits_dev(float v) {
  uint32_t u = __float_as_uint(v);
  return ((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16) & 0xFFFFu;
}

__global__ void rtn_kernel(const float* __restrict__ w, int64_t rows, int64_t cols, const uint32_t* mm_in,
                           uint8_t* codes, uint32_t* minmax) {
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const float* wr = w + r * cols;
  float mn = INFINITY, mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) {
    const float v = wr[i];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
  __shared__ float smn[32], smx[32];
  for (int d = 16; d > 0; d >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(FULL_MASK, mn, d));
    mx = fmaxf(mx, __shfl_xor_sync(FULL_MASK, mx, d));
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  mn = smn[0];
  mx = smx[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
    mn = fminf(mn, smn[i]);
    mx = fmaxf(mx, smx[i]);
  }
  uint32_t bmn = f32_to_bf16_bits_dev(mn), bmx = f32_to_bf16_bits_dev(mx);
  if (mm_in) {  // caller-provided grid (QuantGrid.minmax_bits, quantize.py:80-84)
    bmn = mm_in[r] & 0xFFFFu;
    bmx = mm_in[r] >> 16;
  }
  if (threadIdx.x == 0) minmax[r] = bmn | (bmx << 16);
  double lv[3] = {0.0, (double)__uint_as_float(bmn << 16), (double)__uint_as_float(bmx << 16)};
  // candidate order: ascending |level|, stable in code order
  int ord[3] = {0, 1, 2};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b + 1 < 3 - a; ++b)
      if (fabs(lv[ord[b + 1]]) < fabs(lv[ord[b]])) {
        int t = ord[b];
        ord[b] = ord[b + 1];
        ord[b + 1] = t;
      }
  for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) {
    const double v = (double)wr[i];
    int best = ord[0];
    double bd = fabs(v - lv[ord[0]]);
    for (int c = 1; c < 3; ++c) {
      const double d = fabs(v - lv[ord[c]]);
      if (d < bd) {
        bd = d;
        best = ord[c];
      }
    }
    codes[r * cols + i] = (uint8_t)best;
  }
}

// ================================================================ MoE planner
// Routed-expert dispatcher: stable counting sort of top-1 assignments (token
// order within an expert = buffer order, pipeline.py:86-90) and emission of
// the grouped work units of the wi and wo passes. One CTA.
__global__ void __launch_bounds__(1024) moe_plan_kernel(const int32_t* __restrict__ assign, int T, int E,
                                                        int rows_wi, int rows_wo, int rpu_wi, int rpu_wo,
                                                        int max_units, qmoe_unit* units_wi, qmoe_unit* units_wo,
                                                        int32_t* n_units, int32_t* cnt_out, int32_t* order) {
  extern __shared__ int32_t sh[];
  int32_t* cnt = sh;            // E
  int32_t* start = sh + E;      // E
  int32_t* fill = sh + 2 * E;   // E
  int32_t* uoff = sh + 3 * E;   // E + 1 (units per expert, scanned)
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = fill[e] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int e = assign[t];
    if (e >= 0 && e < E) atomicAdd(&cnt[e], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, u = 0;
    const int nblk_wi = (rows_wi + rpu_wi - 1) / rpu_wi;
    for (int e = 0; e < E; ++e) {
      start[e] = a;
      a += cnt[e];
      uoff[e] = u;
      u += ((cnt[e] + QMOE_NT_MAX - 1) / QMOE_NT_MAX) * nblk_wi;
    }
    uoff[E] = u;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt_out[e] = cnt[e];
  // stable placement, one warp in token order
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int t0 = 0; t0 < T; t0 += 32) {
      const int t = t0 + lane;
      const bool act = t < T;
      const int e = act ? assign[t] : -1;
      const bool ok = act && e >= 0 && e < E;
      const unsigned peers = __match_any_sync(FULL_MASK, ok ? e : -1);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      const int leader = __ffs(peers) - 1;
      int basev = 0;
      if (ok && lane == leader) {
        basev = fill[e];
        fill[e] = basev + __popc(peers);
      }
      basev = __shfl_sync(FULL_MASK, basev, leader);
      if (ok) order[start[e] + basev + rank] = t;
      __syncwarp();
    }
  }
  __syncthreads();
  // units: expert-major, then token chunk, then row block
  const int nblk_wi = (rows_wi + rpu_wi - 1) / rpu_wi;
  const int nblk_wo = (rows_wo + rpu_wo - 1) / rpu_wo;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int c = cnt[e];
    if (!c) continue;
    const int nch = (c + QMOE_NT_MAX - 1) / QMOE_NT_MAX;
    const int ubase_wi = uoff[e];
    const int ubase_wo = (uoff[e] / nblk_wi) * nblk_wo;
    for (int ch = 0; ch < nch; ++ch) {
      qmoe_unit U;
      U.ntok = min(QMOE_NT_MAX, c - ch * QMOE_NT_MAX);
      for (int q = 0; q < QMOE_NT_MAX; ++q) U.tok[q] = order[start[e] + ch * QMOE_NT_MAX + min(q, U.ntok - 1)];
      U.mat = 2 * e;
      for (int b = 0; b < nblk_wi; ++b) {
        const int ui = ubase_wi + ch * nblk_wi + b;
        if (ui < max_units) {
          U.row0 = b * rpu_wi;
          U.row1 = min(rows_wi, U.row0 + rpu_wi);
          units_wi[ui] = U;
        }
      }
      U.mat = 2 * e + 1;
      for (int b = 0; b < nblk_wo; ++b) {
        const int ui = ubase_wo + ch * nblk_wo + b;
        if (ui < max_units) {
          U.row0 = b * rpu_wo;
          U.row1 = min(rows_wo, U.row0 + rpu_wo);
          units_wo[ui] = U;
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    const int chunks = uoff[E] / nblk_wi;
    n_units[0] = min(uoff[E], max_units);
    n_units[1] = min(chunks * nblk_wo, max_units);
    n_units[2] = (uoff[E] > max_units || chunks * nblk_wo > max_units) ? 1 : 0;  // overflow flag
  }
}

// ---------------------------------------------------------------- launch helpers
constexpr int GROUPED_THREADS = 512;

int stage_bytes(int max_cols, int nt) { return (max_cols + 32) * nt * 4; }

// Shared-memory table size: the hot prefix of the entry table that fits beside
// the x staging buffer, capped by `want` (small launches stage less).
int pick_hot(const qmoe_dict* d, int x_bytes, int want) {
  int budget = d->max_smem_optin - x_bytes - 1024;
  int h = budget / 4;
  h = std::min(h, want);
  h = std::min(h, QMOE_DICT_SIZE);
  h &= ~1023;
  return std::max(h, 0);
}

int launch_grouped(const qmoe_dict* d, GroupedParams& P, int max_cols, int nt, int hot_want, int grid,
                   cudaStream_t st) {
  const int xb = stage_bytes(max_cols, nt);
  P.max_cols = max_cols;
  P.H = d->sparse_ok ? pick_hot(d, xb, hot_want) : 0;
  const size_t smem = (size_t)P.H * 4 + xb;
  if (smem > (size_t)d->max_smem_optin)
    return qmoe::fail(QMOE_EUNSUPPORTED, "cols too large for the shared-memory x staging buffer");
  if (d->sparse_ok) {
    CK(cudaFuncSetAttribute(grouped_matvec_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
       "cudaFuncSetAttribute");
    grouped_matvec_kernel<true><<<grid, GROUPED_THREADS, smem, st>>>(P);
  } else {
    CK(cudaFuncSetAttribute(grouped_matvec_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
       "cudaFuncSetAttribute");
    grouped_matvec_kernel<false><<<grid, GROUPED_THREADS, smem, st>>>(P);
  }
  CK(cudaGetLastError(), "grouped_matvec_kernel launch");
  return QMOE_OK;
}

bool bad_dict(const qmoe_dict* d) { return d == nullptr || d->d_stab == nullptr; }

}  // namespace

// ===================================================================== C ABI
extern "C" {

int qmoe_dict_create(const uint32_t* h_words, uint64_t hash64, int device, qmoe_dict_t* out) {
  if (!h_words || !out) return qmoe::fail(QMOE_EINVAL, "null argument");
  *out = nullptr;
  std::vector<uint32_t> stab(QMOE_DICT_SIZE);
  std::vector<uint8_t> len(QMOE_DICT_SIZE);
  std::vector<int32_t> next(size_t(QMOE_DICT_SIZE + 1) * 9), ent(QMOE_DICT_SIZE + 1);
  int max_nz = 0;
  int rc = qmoe::derive_tables(h_words, stab.data(), len.data(), &max_nz);
  if (rc) return rc;
  rc = qmoe::build_trie(h_words, next.data(), ent.data());
  if (rc) return rc;
  CK(cudaSetDevice(device), "cudaSetDevice");
  qmoe_dict* d = new qmoe_dict();
  d->device = device;
  d->hash64 = hash64;
  d->max_nz = max_nz;
  d->sparse_ok = max_nz <= 3;
  cudaDeviceGetAttribute(&d->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&d->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  cudaError_t e;
  if ((e = cudaMalloc(&d->d_words, QMOE_DICT_SIZE * 8)) != cudaSuccess ||
      (e = cudaMalloc(&d->d_stab, QMOE_DICT_SIZE * 4)) != cudaSuccess ||
      (e = cudaMalloc(&d->d_len, QMOE_DICT_SIZE)) != cudaSuccess ||
      (e = cudaMalloc(&d->d_next, next.size() * 4)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_words, h_words, QMOE_DICT_SIZE * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_stab, stab.data(), QMOE_DICT_SIZE * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_len, len.data(), QMOE_DICT_SIZE, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_next, next.data(), next.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) {
    qmoe_dict_destroy(d);
    return cuda_fail(e, "dictionary upload");
  }
  *out = d;
  return QMOE_OK;
}

int qmoe_dict_destroy(qmoe_dict_t d) {
  if (!d) return QMOE_OK;
  cudaFree(d->d_words);
  cudaFree(d->d_stab);
  cudaFree(d->d_len);
  cudaFree(d->d_next);
  delete d;
  return QMOE_OK;
}

int qmoe_dict_info(qmoe_dict_t d, uint64_t* hash64, int* max_nonzeros, int* sparse_path) {
  if (!d) return qmoe::fail(QMOE_EINVAL, "null dictionary");
  if (hash64) *hash64 = d->hash64;
  if (max_nonzeros) *max_nonzeros = d->max_nz;
  if (sparse_path) *sparse_path = d->sparse_ok;
  return QMOE_OK;
}

int qmoe_validate_rows(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, int64_t rows, int64_t cols,
                       int32_t* d_bad, void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || !d_bad) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows == 0) return QMOE_OK;
  const int64_t blocks = std::min<int64_t>((rows + 7) / 8, 4 * d->num_sms);
  validate_rows_kernel<<<(int)blocks, 256, 0, S(stream)>>>(d->d_len, d_cw, d_row_off, rows, cols, d_bad);
  CK(cudaGetLastError(), "validate_rows_kernel");
  return QMOE_OK;
}

int qmoe_decompress(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, int64_t rows, int64_t cols,
                    uint8_t* d_out, int32_t* d_bad, void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || cols % 2 || !d_bad) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows == 0) return QMOE_OK;
  cudaStream_t st = S(stream);
  if (cols) CK(cudaMemsetAsync(d_out, 0, (size_t)rows * cols, st), "memset");
  // Decompress is write-bound (rows*cols output bytes per ~2 bits read): a
  // modest hot table keeps the per-CTA table fill cheap.
  const int H = d->sparse_ok ? std::min(32768, (int)std::max<int64_t>(1024, (rows * cols / 16 / d->num_sms) & ~1023)) : 0;
  const int64_t blocks = std::min<int64_t>((rows + 15) / 16, d->num_sms);
  const size_t smem = (size_t)H * 4;
  if (d->sparse_ok) {
    CK(cudaFuncSetAttribute(decompress_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    decompress_kernel<true><<<(int)blocks, 512, smem, st>>>(d->d_stab, d->d_words, H, d_cw, d_row_off, rows, cols,
                                                            d_out, d_bad);
  } else {
    decompress_kernel<false><<<(int)blocks, 512, 0, st>>>(d->d_stab, d->d_words, 0, d_cw, d_row_off, rows, cols,
                                                          d_out, d_bad);
  }
  CK(cudaGetLastError(), "decompress_kernel");
  return QMOE_OK;
}

static int fused_common(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, const uint32_t* d_mm,
                        int64_t rows, int64_t cols, const void* d_x, int x_dtype, int64_t ntok, int64_t ldx,
                        float* d_y, int64_t ldy, int32_t* d_bad, void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || cols % 2 || ntok < 0 || (x_dtype != QMOE_X_F32 && x_dtype != QMOE_X_BF16))
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows > INT32_MAX || cols > INT32_MAX) return qmoe::fail(QMOE_EINVAL, "matrix too large");
  if (rows == 0 || ntok == 0) return QMOE_OK;
  GroupedParams P{};
  P.stab = d->d_stab;
  P.words = d->d_words;
  P.units = nullptr;
  P.single = qmoe_matrix{d_cw, d_row_off, d_mm, (int32_t)rows, (int32_t)cols};
  P.ntok_single = ntok;
  P.x = d_x;
  P.x_dtype = x_dtype;
  P.ldx = ldx;
  P.x_relu = 0;
  P.y = d_y;
  P.ldy = ldy;
  P.bad = d_bad;
  // Work split: ~32 rows per unit; grid no larger than the unit count so tiny
  // matrices do not pay a full-chip table fill.
  P.rows_per_unit = 32;
  const int64_t nblk = (rows + P.rows_per_unit - 1) / P.rows_per_unit;
  const int64_t units = nblk * ((ntok + QMOE_NT_MAX - 1) / QMOE_NT_MAX);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, d->num_sms));
  const int nt = ntok == 1 ? 1 : (ntok == 2 ? 2 : 4);
  return launch_grouped(d, P, (int)cols, nt, QMOE_DICT_SIZE, grid, S(stream));
}

int qmoe_fused_matvec(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, const uint32_t* d_mm,
                      int64_t rows, int64_t cols, const void* d_x, int x_dtype, float* d_y, int32_t* d_bad,
                      void* stream) {
  return fused_common(d, d_cw, d_row_off, d_mm, rows, cols, d_x, x_dtype, 1, cols, d_y, rows, d_bad, stream);
}

int qmoe_fused_matmat(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, const uint32_t* d_mm,
                      int64_t rows, int64_t cols, const void* d_x, int x_dtype, int64_t ntok, int64_t ldx,
                      float* d_y, int64_t ldy, int32_t* d_bad, void* stream) {
  if (ldx < cols || ldy < rows) return qmoe::fail(QMOE_EINVAL, "leading dimension too small");
  return fused_common(d, d_cw, d_row_off, d_mm, rows, cols, d_x, x_dtype, ntok, ldx, d_y, ldy, d_bad, stream);
}

int qmoe_grouped_matvec(qmoe_dict_t d, const qmoe_matrix* d_mats, const qmoe_unit* d_units, const int32_t* d_n_units,
                        int32_t max_units, int32_t max_cols, const void* d_x, int x_dtype, int64_t ldx, int x_relu,
                        float* d_y, int64_t ldy, int32_t* d_bad, void* stream) {
  if (bad_dict(d) || !d_mats || !d_units || !d_n_units || max_units < 0 || max_cols <= 0 ||
      (x_dtype != QMOE_X_F32 && x_dtype != QMOE_X_BF16))
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (max_units == 0) return QMOE_OK;
  GroupedParams P{};
  P.stab = d->d_stab;
  P.words = d->d_words;
  P.mats = d_mats;
  P.units = d_units;
  P.n_units = d_n_units;
  P.max_units = max_units;
  P.x = d_x;
  P.x_dtype = x_dtype;
  P.ldx = ldx;
  P.x_relu = x_relu;
  P.y = d_y;
  P.ldy = ldy;
  P.bad = d_bad;
  return launch_grouped(d, P, max_cols, QMOE_NT_MAX, QMOE_DICT_SIZE, d->num_sms, S(stream));
}

int qmoe_paper_matvec(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, const uint32_t* d_mm,
                      int64_t rows, int64_t cols, const void* d_x, int x_dtype, float* d_y, int32_t* d_trace,
                      void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || (x_dtype != QMOE_X_F32 && x_dtype != QMOE_X_BF16))
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows == 0) return QMOE_OK;
  const size_t smem = (size_t)(cols + 32) * 4 + 3 * 32 * PAPER_WARPS * 4 + PAPER_WARPS * 32 * 2;
  if (smem > (size_t)d->max_smem_optin) return qmoe::fail(QMOE_EUNSUPPORTED, "cols too large");
  CK(cudaFuncSetAttribute(paper_matvec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
  // one CTA per SM with min(rows, 32) warps
  const int grid = (int)std::min<int64_t>(d->num_sms, (rows + PAPER_WARPS - 1) / PAPER_WARPS);
  paper_matvec_kernel<<<grid, PAPER_WARPS * 32, smem, S(stream)>>>(d->d_words, d_cw, d_row_off, d_mm, (int)rows,
                                                                   (int)cols, d_x, x_dtype, d_y, d_trace);
  CK(cudaGetLastError(), "paper_matvec_kernel");
  return QMOE_OK;
}

int qmoe_encode_count(qmoe_dict_t d, const uint8_t* d_codes, int64_t rows, int64_t cols, int32_t* d_counts,
                      void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || cols % 2) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows == 0) return QMOE_OK;
  encode_kernel<false><<<(int)((rows + 127) / 128), 128, 0, S(stream)>>>(d->d_next, d_codes, rows, cols, d_counts,
                                                                         nullptr, nullptr);
  CK(cudaGetLastError(), "encode_count");
  return QMOE_OK;
}

int qmoe_encode_emit(qmoe_dict_t d, const uint8_t* d_codes, int64_t rows, int64_t cols, const int32_t* d_row_off,
                     uint16_t* d_cw, void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || cols % 2) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows == 0) return QMOE_OK;
  encode_kernel<true><<<(int)((rows + 127) / 128), 128, 0, S(stream)>>>(d->d_next, d_codes, rows, cols, nullptr,
                                                                        d_row_off, d_cw);
  CK(cudaGetLastError(), "encode_emit");
  return QMOE_OK;
}

int qmoe_exclusive_scan(const int32_t* d_in, int64_t n, int32_t* d_out, void* stream) {
  if (n < 0 || !d_out) return qmoe::fail(QMOE_EINVAL, "bad argument");
  exclusive_scan_kernel<<<1, 1024, 0, S(stream)>>>(d_in, n, d_out);
  CK(cudaGetLastError(), "exclusive_scan");
  return QMOE_OK;
}

int qmoe_rtn_quantize(const float* d_w, int64_t rows, int64_t cols, const uint32_t* d_mm_in, uint8_t* d_codes,
                      uint32_t* d_mm, void* stream) {
  if (rows < 0 || cols < 1) return qmoe::fail(QMOE_EINVAL, "weights must be a non-empty 2d array");
  if (rows == 0) return QMOE_OK;
  rtn_kernel<<<(int)rows, 256, 0, S(stream)>>>(d_w, rows, cols, d_mm_in, d_codes, d_mm);
  CK(cudaGetLastError(), "rtn_kernel");
  return QMOE_OK;
}

int qmoe_moe_plan(const int32_t* d_assign, int32_t T, int32_t E, int32_t rows_wi, int32_t rows_wo,
                  int32_t rpu_wi, int32_t rpu_wo, int32_t max_units, qmoe_unit* d_units_wi, qmoe_unit* d_units_wo,
                  int32_t* d_n_units, int32_t* d_expert_count, int32_t* d_order, void* stream) {
  if (T < 0 || E < 1 || rows_wi < 1 || rows_wo < 1 || rpu_wi < 1 || rpu_wo < 1 || max_units < 0)
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  const size_t smem = (size_t)(4 * E + 1) * 4;
  if (smem > 200 * 1024) return qmoe::fail(QMOE_EUNSUPPORTED, "too many experts");
  CK(cudaFuncSetAttribute(moe_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
  moe_plan_kernel<<<1, 1024, smem, S(stream)>>>(d_assign, T, E, rows_wi, rows_wo, rpu_wi, rpu_wo, max_units,
                                                 d_units_wi, d_units_wo, d_n_units, d_expert_count, d_order);
  CK(cudaGetLastError(), "moe_plan_kernel");
  return QMOE_OK;
}

}  // extern "C"
