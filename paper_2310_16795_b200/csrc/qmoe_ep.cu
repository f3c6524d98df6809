// Expert-parallel exchange helpers: the fixed-slot
// dispatch / combine of ep.ExpertParallelMoE as two small kernels instead of a
// chain of framework ops, so an EP step is: slots -> scatter -> NCCL
// all-to-all (x, ids) -> fused local step -> all-to-all (y) -> gather.
//
//  qmoe_ep_slots     one CTA: token t with expert id a in [0, E) goes to rank
//                    d = a / (E / world) at slot d * C + (stable rank of t among
//                    the tokens bound for d) (pipeline.py:86-90 buffer order),
//                    C = slots per destination (the layer's token capacity, the
//                    same on every rank, so every all-to-all has equal splits);
//                    id_send gets the rank-local id there, -1 in empty slots.
//  qmoe_ep_rows      row moves by an index: scatter dst[idx[i]] = src[i] or
//                    gather dst[i] = src[idx[i]] (zero row for idx -1).
//  qmoe_ep_combine   gather of the returned bf16 expert rows into f32 output
//                    rows (exact: the expert outputs are bf16-rounded values),
//                    zero rows for tokens without an expert.

#include <cuda_runtime.h>
#include <stdint.h>

#include "qmoe.h"
#include "qmoe_internal.h"

namespace {

constexpr int EP_THREADS = 1024;
constexpr int EP_MAXW = 64;

__global__ void __launch_bounds__(EP_THREADS) ep_slots_kernel(const int32_t* __restrict__ assign, int T, int E,
                                                               int world, int C, int32_t* slot, int32_t* id_send,
                                                               int32_t* send_counts) {
  __shared__ int wcnt[EP_THREADS / 32][EP_MAXW];  // per warp, per destination
  __shared__ int base[EP_MAXW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = E / world;
  for (int i = tid; i < world * C; i += EP_THREADS) id_send[i] = -1;
  if (tid < world) base[tid] = 0;
  __syncthreads();
  for (int t0 = 0; t0 < T; t0 += EP_THREADS) {
    const int t = t0 + tid;
    const int a = t < T ? assign[t] : -1;
    const bool ok = t < T && a >= 0 && a < E;
    const int d = ok ? a / per : -1;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    for (int k = lane; k < world; k += 32) wcnt[warp][k] = 0;
    __syncwarp();
    if (ok && (__ffs(peers) - 1) == lane) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (tid < world) {  // exclusive scan over the warps of this tile, per destination
      int run = base[tid];
      for (int w = 0; w < EP_THREADS / 32; ++w) {
        const int c = wcnt[w][tid];
        wcnt[w][tid] = run;
        run += c;
      }
      base[tid] = run;
    }
    __syncthreads();
    if (t < T) {
      const int s = ok ? d * C + wcnt[warp][d] + rank : -1;
      slot[t] = s;
      if (ok) id_send[s] = a - d * per;
    }
    __syncthreads();
  }
  if (send_counts && tid < world) send_counts[tid] = base[tid];
}

__global__ void ep_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int n, int v16,
                               const int32_t* __restrict__ idx, int scatter) {
  // one warp per row, 16-byte vectors
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int j = idx[row];
  if (scatter) {
    if (j < 0) return;
    for (int v = lane; v < v16; v += 32) dst[(int64_t)j * v16 + v] = src[(int64_t)row * v16 + v];
  } else {
    for (int v = lane; v < v16; v += 32)
      dst[(int64_t)row * v16 + v] = j >= 0 ? src[(int64_t)j * v16 + v] : make_uint4(0u, 0u, 0u, 0u);
  }
}

__global__ void ep_combine_kernel(const uint16_t* __restrict__ src, float* __restrict__ dst, int n, int d,
                                  const int32_t* __restrict__ idx) {
  // one warp per output row: dst[i] = f32(src[idx[i]]) (bf16 -> f32 exact)
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int j = idx[row];
  for (int v = lane; v < d; v += 32)
    dst[(int64_t)row * d + v] = j >= 0 ? __uint_as_float(uint32_t(src[(int64_t)j * d + v]) << 16) : 0.f;
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" int qmoe_ep_slots(const int32_t* d_assign, int32_t T, int32_t E, int32_t world, int32_t slots_per_rank,
                             int32_t* d_slot, int32_t* d_id_send, int32_t* d_send_counts, void* stream) {
  if (!d_assign || T < 0 || E < 1 || world < 1 || world > EP_MAXW || E % world || !d_slot || !d_id_send ||
      slots_per_rank < T)
    return qmoe::fail(QMOE_EINVAL, "bad argument (1 <= world <= 64, world divides E, T <= slots_per_rank)");
  ep_slots_kernel<<<1, EP_THREADS, 0, S(stream)>>>(d_assign, T, E, world, slots_per_rank, d_slot, d_id_send,
                                                   d_send_counts);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QMOE_OK : qmoe::fail(QMOE_ECUDA, cudaGetErrorString(e));
}

extern "C" int qmoe_ep_rows(const void* d_src, void* d_dst, int32_t n_rows, int64_t row_bytes, const int32_t* d_index,
                            int scatter, void* stream) {
  if (n_rows == 0) return QMOE_OK;
  if (!d_src || !d_dst || !d_index || n_rows < 0 || row_bytes <= 0 || row_bytes % 16 ||
      (reinterpret_cast<uintptr_t>(d_src) & 15) || (reinterpret_cast<uintptr_t>(d_dst) & 15))
    return qmoe::fail(QMOE_EINVAL, "bad argument (16-byte aligned rows)");
  const int wpb = 8;
  ep_rows_kernel<<<(n_rows + wpb - 1) / wpb, wpb * 32, 0, S(stream)>>>(
      reinterpret_cast<const uint4*>(d_src), reinterpret_cast<uint4*>(d_dst), n_rows, (int)(row_bytes / 16), d_index,
      scatter);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QMOE_OK : qmoe::fail(QMOE_ECUDA, cudaGetErrorString(e));
}

extern "C" int qmoe_ep_combine(const uint16_t* d_src_bf16, float* d_dst, int32_t n_rows, int32_t d,
                               const int32_t* d_index, void* stream) {
  if (n_rows == 0) return QMOE_OK;
  if (!d_src_bf16 || !d_dst || !d_index || n_rows < 0 || d <= 0) return qmoe::fail(QMOE_EINVAL, "bad argument");
  const int wpb = 8;
  ep_combine_kernel<<<(n_rows + wpb - 1) / wpb, wpb * 32, 0, S(stream)>>>(d_src_bf16, d_dst, n_rows, d, d_index);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QMOE_OK : qmoe::fail(QMOE_ECUDA, cudaGetErrorString(e));
}
