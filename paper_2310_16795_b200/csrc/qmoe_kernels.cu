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

#include "qmoe_device.cuh"


namespace {
using namespace qmoe_dev;

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

// ================================================================ decompress
// _decode_range (codec.py:158-172) into a zero-initialised (rows, cols) u8
// buffer: only non-zero codes are stored (sparse path) or every value of the
// entry (general path). Same warp-per-row lane-segment schedule.
template <int K>
__device__ __forceinline__ void dseg_sparse(const uint16_t* __restrict__ cwp, int cnt, int lane,
                                            const SparseTab& tab, uint8_t* out, int64_t cols, int& base) {
  // matvec-format entries (esz 4 variant): field / 4 = position in the entry
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
      if ((t[k] >> (26 + j)) & 1u) {
        const int c = off + int(((t[k] >> (5 + 7 * j)) & 0x7Fu) >> 2);
        if (c < cols) out[c] = ((t[k] >> (29 + j)) & 1u) ? 2 : 1;
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
// order within an expert = buffer order, pipeline.py:86-90) and the run lists
// of the wi and wo passes (one run per expert token chunk, all rows). One CTA
// of 1024 threads; per-expert prefixes by a block scan, so the cost is
// O(E/1024 + T/32) steps.
__device__ __forceinline__ int run_tasks_dev(int rows, int lg) { return ((rows << lg) + 31) >> 5; }

__device__ __forceinline__ int4 block_scan_excl(int4 v, int4* wsum, int4* total) {
  // exclusive scan of int4 values over the 1024 threads (thread order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int4 incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int4 o;
    o.x = __shfl_up_sync(FULL_MASK, incl.x, d);
    o.y = __shfl_up_sync(FULL_MASK, incl.y, d);
    o.z = __shfl_up_sync(FULL_MASK, incl.z, d);
    o.w = __shfl_up_sync(FULL_MASK, incl.w, d);
    if (lane >= d) {
      incl.x += o.x;
      incl.y += o.y;
      incl.z += o.z;
      incl.w += o.w;
    }
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int4 w = wsum[lane];
    int4 wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int4 o;
      o.x = __shfl_up_sync(FULL_MASK, wi.x, d);
      o.y = __shfl_up_sync(FULL_MASK, wi.y, d);
      o.z = __shfl_up_sync(FULL_MASK, wi.z, d);
      o.w = __shfl_up_sync(FULL_MASK, wi.w, d);
      if (lane >= d) {
        wi.x += o.x;
        wi.y += o.y;
        wi.z += o.z;
        wi.w += o.w;
      }
    }
    wsum[lane] = make_int4(wi.x - w.x, wi.y - w.y, wi.z - w.z, wi.w - w.w);
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const int4 b = wsum[warp];
  return make_int4(b.x + incl.x - v.x, b.y + incl.y - v.y, b.z + incl.z - v.z, b.w + incl.w - v.w);
}

// lanes per row of a run: the override, bounded by the checkpoint
// granularity the matrix stores (M.lg)
__device__ __forceinline__ int plan_lg(const qmoe_matrix& M, int lg_over) {
  if (lg_over < 0) return M.lg;
  return min(lg_over, M.lg);
}

__global__ void __launch_bounds__(1024) moe_plan_kernel(const int32_t* __restrict__ assign, int T, int E,
                                                        const qmoe_matrix* __restrict__ mats, int ntu, int lg_wi,
                                                        int lg_wo, int max_runs,
                                                        qmoe_work* runs_wi, qmoe_work* runs_wo, int32_t* n_out,
                                                        int32_t* cnt_out, int32_t* order, int stage_ids) {
  extern __shared__ int32_t sh[];
  int32_t* cnt = sh;             // E: tokens per expert (then fill cursor)
  int32_t* start = sh + E;       // E: first slot of expert e in order[]
  int32_t* choff = sh + 2 * E;   // E + 1: token chunks before expert e
  int32_t* twi = sh + 3 * E + 1; // E: wi tasks before expert e
  int32_t* two = sh + 4 * E + 1; // E: wo tasks before expert e
  int32_t* ids = sh + 5 * E + 1;  // T (when staged): the ids, read once from global
  __shared__ int4 wsum[32];
  __shared__ int4 total;
  const bool staged = stage_ids != 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int e = assign[t];
    if (staged) ids[t] = e;
    if (e >= 0 && e < E) atomicAdd(&cnt[e], 1);
  }
  __syncthreads();
  // per-thread contiguous expert slice, block scan of (tokens, chunks, wi tasks, wo tasks)
  const int per = (E + blockDim.x - 1) / blockDim.x;
  const int e0 = min(E, (int)threadIdx.x * per), e1 = min(E, e0 + per);
  int4 loc = make_int4(0, 0, 0, 0);
  for (int e = e0; e < e1; ++e) {
    const int c = cnt[e], nch = (c + ntu - 1) / ntu;
    loc.x += c;
    loc.y += nch;
    if (nch) {
      loc.z += nch * run_tasks_dev(mats[2 * e].rows, plan_lg(mats[2 * e], lg_wi));
      loc.w += nch * run_tasks_dev(mats[2 * e + 1].rows, plan_lg(mats[2 * e + 1], lg_wo));
    }
  }
  int4 base = block_scan_excl(loc, wsum, &total);
  for (int e = e0; e < e1; ++e) {
    const int c = cnt[e], nch = (c + ntu - 1) / ntu;
    start[e] = base.x;
    choff[e] = base.y;
    twi[e] = base.z;
    two[e] = base.w;
    base.x += c;
    base.y += nch;
    if (nch) {
      base.z += nch * run_tasks_dev(mats[2 * e].rows, plan_lg(mats[2 * e], lg_wi));
      base.w += nch * run_tasks_dev(mats[2 * e + 1].rows, plan_lg(mats[2 * e + 1], lg_wo));
    }
    cnt_out[e] = c;
    cnt[e] = 0;  // becomes the fill cursor
  }
  if (threadIdx.x == 0) choff[E] = total.y;
  __syncthreads();
  // stable placement, one warp walking the tokens in buffer order
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int t0 = 0; t0 < T; t0 += 32) {
      const int t = t0 + lane;
      const int e = t < T ? (staged ? ids[t] : assign[t]) : -1;
      const bool ok = t < T && e >= 0 && e < E;
      const unsigned peers = __match_any_sync(FULL_MASK, ok ? e : -1);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      const int leader = __ffs(peers) - 1;
      int basev = 0;
      if (ok && lane == leader) {
        basev = cnt[e];
        cnt[e] = basev + __popc(peers);
      }
      basev = __shfl_sync(FULL_MASK, basev, leader);
      if (ok) order[start[e] + basev + rank] = t;
      __syncwarp();
    }
  }
  __syncthreads();
  const int nchunks = min(choff[E], max_runs);
  for (int i = threadIdx.x; i < nchunks; i += blockDim.x) {
    int lo = 0, hi = E - 1;  // expert owning chunk i: last e with choff[e] <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (choff[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const int e = lo, ch = i - choff[e];
    const int c = cnt[e];  // == tokens of e after placement
    qmoe_work U;
    U.ntok = min(ntu, c - ch * ntu);
    for (int q = 0; q < QMOE_NT_MAX; ++q) U.tok[q] = order[start[e] + ch * ntu + min(q, U.ntok - 1)];
    for (int pass = 0; pass < 2; ++pass) {
      const qmoe_matrix M = mats[2 * e + pass];
      U.cw = M.cw;
      U.row_off = M.row_off;
      U.row_minmax = M.row_minmax;
      U.ck = M.ck;
      U.row_id = M.row_id;
      const int rlg = plan_lg(M, pass ? lg_wo : lg_wi);
      U.lg = rlg | (M.lg << 8);  // checkpoint stride in bits 8-15
      U.cols = M.cols;
      U.row0 = 0;
      U.row1 = M.rows;
      U.task0 = (pass ? two[e] : twi[e]) + ch * run_tasks_dev(M.rows, rlg);
      (pass ? runs_wo : runs_wi)[i] = U;
    }
  }
  if (threadIdx.x == 0) {
    n_out[0] = nchunks;
    n_out[1] = choff[E] <= max_runs ? total.z : (nchunks ? 0 : 0);
    n_out[2] = nchunks;
    n_out[3] = choff[E] <= max_runs ? total.w : 0;
  }
}

// ================================================================ codebook
// Frequency codebook (kernel-private re-indexing, include/qmoe.h).
__global__ void histogram_kernel(const uint16_t* __restrict__ cw, int64_t n, uint32_t* counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(counts + __ldg(cw + i), 1u);
}
__global__ void remap_kernel(const uint16_t* __restrict__ in, int64_t n, const uint16_t* __restrict__ rank_of,
                             uint16_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldg(rank_of + in[i]);
}

// ================================================================ checkpoints
// Row-segment checkpoints (include/qmoe.h qmoe_checkpoints): thread per row
// walks the row's codewords once, summing entry lengths, and records the
// column at each segment start s + (j*n >> lg).
__global__ void checkpoints_kernel(const uint32_t* __restrict__ tab, const uint16_t* __restrict__ cw,
                                   const int32_t* __restrict__ row_off, int64_t rows, int64_t cols, int lg,
                                   uint16_t* ck, int32_t* bad) {
  // thread per row: the start column of segments 1 .. G-1 (qmoe_device.cuh
  // seg_start: group-aligned boundaries)
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int G = 1 << lg;
  const int s = __ldg(row_off + r), e = __ldg(row_off + r + 1);
  int j = 1, next = G > 1 ? seg_start(s, e, 1, lg) : e;
  int off = 0;
  for (int k = s; k < e; ++k) {
    while (j < G && k == next) {
      ck[r * (G - 1) + j - 1] = (uint16_t)min(off, 65535);
      ++j;
      next = seg_start(s, e, j, lg);
    }
    off += int(__ldg(tab + __ldg(cw + k)) & 31u);
  }
  while (j < G) {  // empty tail segments
    ck[r * (G - 1) + j - 1] = (uint16_t)min(off, 65535);
    ++j;
  }
  if (off != cols && bad) {
    atomicAdd(bad, 1);
    atomicMin(bad + 1, (int)r);
  }
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
  std::vector<uint32_t> mtab(2 * (size_t)qmoe::MT_STRIDE);
  qmoe::derive_matvec_tables(stab.data(), mtab.data());
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
      (e = cudaMalloc(&d->d_mtab, mtab.size() * 4)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_mtab, mtab.data(), mtab.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMalloc(&d->d_next, next.size() * 4)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_words, h_words, QMOE_DICT_SIZE * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_stab, stab.data(), QMOE_DICT_SIZE * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_len, len.data(), QMOE_DICT_SIZE, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(d->d_next, next.data(), next.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) {
    qmoe_dict_destroy(d);
    return cuda_fail(e, "dictionary upload");
  }
  d->h_mtab = std::move(mtab);
  *out = d;
  return QMOE_OK;
}

int qmoe_dict_destroy(qmoe_dict_t d) {
  if (!d) return QMOE_OK;
  cudaFree(d->d_words);
  cudaFree(d->d_stab);
  cudaFree(d->d_len);
  cudaFree(d->d_mtab);
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

int qmoe_decompress(qmoe_dict_t d, const uint32_t* d_table, const uint16_t* d_cw, const int32_t* d_row_off,
                    int64_t rows, int64_t cols, uint8_t* d_out, int32_t* d_bad, void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || cols % 2 || !d_bad) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows == 0) return QMOE_OK;
  if (d_table && !d->sparse_ok) return qmoe::fail(QMOE_EUNSUPPORTED, "codebooks need a <=3-non-zero dictionary");
  cudaStream_t st = S(stream);
  if (cols) CK(cudaMemsetAsync(d_out, 0, (size_t)rows * cols, st), "memset");
  // Decompress is write-bound (rows*cols output bytes per ~2 bits read): a
  // modest hot table keeps the per-CTA table fill cheap.
  const int H = d->sparse_ok ? std::min(32768, (int)std::max<int64_t>(1024, (rows * cols / 16 / d->num_sms) & ~1023)) : 0;
  const int64_t blocks = std::min<int64_t>((rows + 15) / 16, d->num_sms);
  const size_t smem = (size_t)H * 4;
  if (d->sparse_ok) {
    CK(cudaFuncSetAttribute(decompress_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    decompress_kernel<true><<<(int)blocks, 512, smem, st>>>(d_table ? d_table : d->d_mtab, d->d_words, H, d_cw,
                                                            d_row_off, rows, cols, d_out, d_bad);
  } else {
    decompress_kernel<false><<<(int)blocks, 512, 0, st>>>(d->d_stab, d->d_words, 0, d_cw, d_row_off, rows, cols,
                                                          d_out, d_bad);
  }
  CK(cudaGetLastError(), "decompress_kernel");
  return QMOE_OK;
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

int qmoe_moe_plan(const int32_t* d_assign, int32_t T, int32_t E, const qmoe_matrix* d_mats, int32_t ntu,
                  int32_t lg_wi, int32_t lg_wo, int32_t max_runs, qmoe_work* d_runs_wi, qmoe_work* d_runs_wo, int32_t* d_n,
                  int32_t* d_expert_count, int32_t* d_order, void* stream) {
  if (T < 0 || E < 1 || !d_mats || max_runs < T || ntu < 1 || ntu > QMOE_NT_MAX || !d_n || lg_wi > 5 || lg_wo > 5)
    return qmoe::fail(QMOE_EINVAL, "bad argument (max_runs must be >= T)");
  size_t smem = (size_t)(5 * E + 1) * 4;
  if (smem > 200 * 1024) return qmoe::fail(QMOE_EUNSUPPORTED, "too many experts");
  const int stage = smem + (size_t)T * 4 <= 200 * 1024 ? 1 : 0;  // ids in shared memory for the ordered walk
  if (stage) smem += (size_t)T * 4;
  CK(cudaFuncSetAttribute(moe_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
  moe_plan_kernel<<<1, 1024, smem, S(stream)>>>(d_assign, T, E, d_mats, ntu, lg_wi, lg_wo, max_runs, d_runs_wi,
                                                 d_runs_wo, d_n,
                                                 d_expert_count, d_order, stage);
  CK(cudaGetLastError(), "moe_plan_kernel");
  return QMOE_OK;
}

int qmoe_histogram(const uint16_t* d_cw, int64_t n, uint32_t* d_counts, void* stream) {
  if (n < 0 || !d_counts) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (n == 0) return QMOE_OK;
  histogram_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1184), 256, 0, S(stream)>>>(d_cw, n, d_counts);
  CK(cudaGetLastError(), "histogram_kernel");
  return QMOE_OK;
}

int qmoe_codebook_table(qmoe_dict_t d, const uint16_t* h_order, uint32_t* d_table) {
  if (bad_dict(d) || !h_order || !d_table) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (!d->sparse_ok) return qmoe::fail(QMOE_EUNSUPPORTED, "codebooks need a <=3-non-zero dictionary");
  std::vector<uint8_t> seen(QMOE_DICT_SIZE, 0);
  const size_t V = qmoe::MT_STRIDE;
  std::vector<uint32_t> t(2 * V, 0u);
  for (int k = 0; k < QMOE_DICT_SIZE; ++k) {
    const uint16_t c = h_order[k];
    if (seen[c]++) return qmoe::fail(QMOE_EINVAL, "order is not a permutation of the 65536 codewords");
    t[k] = d->h_mtab[c];
    t[V + k] = d->h_mtab[V + c];
  }
  CK(cudaMemcpy(d_table, t.data(), t.size() * 4, cudaMemcpyHostToDevice), "codebook upload");
  return QMOE_OK;
}

int qmoe_remap(const uint16_t* d_in, int64_t n, const uint16_t* d_rank_of, uint16_t* d_out, void* stream) {
  if (n < 0 || !d_rank_of) return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (n == 0) return QMOE_OK;
  remap_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4736), 256, 0, S(stream)>>>(d_in, n, d_rank_of, d_out);
  CK(cudaGetLastError(), "remap_kernel");
  return QMOE_OK;
}

int qmoe_checkpoints(qmoe_dict_t d, const uint32_t* d_table, const uint16_t* d_cw, const int32_t* d_row_off,
                     int64_t rows, int64_t cols, int lg, uint16_t* d_ck, int32_t* d_bad, void* stream) {
  if (bad_dict(d) || rows < 0 || cols < 0 || cols > 65535 || lg < 1 || lg > 5 || !d_ck)
    return qmoe::fail(QMOE_EINVAL, "bad argument (1 <= lg <= 5, cols <= 65535)");
  if (!d->sparse_ok) return qmoe::fail(QMOE_EUNSUPPORTED, "checkpoints need a <=3-non-zero dictionary");
  if (rows == 0) return QMOE_OK;
  checkpoints_kernel<<<(int)((rows + 127) / 128), 128, 0, S(stream)>>>(d_table ? d_table : d->d_mtab, d_cw,
                                                                        d_row_off, rows, cols, lg, d_ck, d_bad);
  CK(cudaGetLastError(), "checkpoints_kernel");
  return QMOE_OK;
}

}  // extern "C"
