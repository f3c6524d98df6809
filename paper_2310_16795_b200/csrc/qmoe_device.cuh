// Device-side declarations shared by the libqmoe CUDA translation units.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
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
  uint32_t* d_mtab = nullptr;    // matvec-format tables: [esz 4 | esz 2] x MT_STRIDE (zero entries from 65536)
  std::vector<uint32_t> h_mtab;  // host copy (codebook construction)
  uint8_t* d_len = nullptr;      // 2n per entry
  int32_t* d_next = nullptr;     // trie next_node (65537, 9)
};

namespace qmoe_dev {

inline int cuda_fail(cudaError_t e, const char* what) {
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

// Row segments of the streaming kernels (kernel-private checkpoints): segment
// j of a row [s, e) split in 2^lg starts at the equal split s + j*n/2^lg
// rounded UP to a multiple of 8 codewords (a 16-byte group of the stream), so
// only a row's first and last groups are shared with neighbouring rows.
// Boundaries nest: seg_start(s, e, j, lg) == seg_start(s, e, 2j, lg + 1).
__device__ __forceinline__ int seg_start(int s, int e, int j, int lg) {
  if (j == 0) return s;
  const int b = (s + ((j * (e - s)) >> lg) + 7) & ~7;
  return b < e ? b : e;
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


}  // namespace qmoe_dev
