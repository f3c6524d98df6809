// Batched-token decode-then-MMA MoE pass (BASELINE
// configs[2]: Switch-large-128 with many tokens per expert).
//
// With t tokens per expert the streaming matvec re-decodes each expert matrix
// ceil(t / 2) times; here every expert row block is decoded ONCE per step into
// a dense bf16 tile in shared memory and multiplied on the tensor cores with
// all of the expert's tokens (up to 64 per block).
//
//   work item   (expert e, 512-row block, token block of <= BN tokens); the
//               persistent grid strides over the items; every CTA derives the
//               item list from the dispatcher's expert counts (qmoe_moe_plan).
//   decode      thread = row: the lane walks its row's codeword stream chunk
//               by chunk (64 columns), zero-fills its 128-byte row of the W
//               tile and stores the <= 3 non-zero bf16 levels of each codeword
//               (entry table of the streaming kernel, hot prefix in shared
//               memory). A codeword straddling the chunk end is revisited by
//               the next chunk. Rows are XOR-swizzled by 16-byte chunk so the
//               MMA operand loads are bank-conflict free.
//   mma         warp w owns rows [32w, 32w+32) — exactly the rows its lanes
//               decoded — x BN tokens: ldmatrix + mma.sync.m16n8k16 bf16 ->
//               fp32 accumulators in registers; the token tile (bf16, from
//               x rows of the expert's tokens) is double-buffered per chunk.
//   epilogue    per (row, token): bf16 RNE once (codec.py:243), y mode as the
//               streaming kernel (relu -> bf16 hidden, or f32 store / add).
//
// Numerics: bf16 x bf16 products are exact in fp32; the accumulation order
// differs from the reference's sgemv (tolerance-level parity, as the
// streaming kernel).
#include <algorithm>
#include <climits>

#include "qmoe_device.cuh"

using namespace qmoe_dev;

namespace {

constexpr int DTHREADS = 512;
constexpr int DWARPS = DTHREADS / 32;
constexpr int BM = DTHREADS;  // rows per item (thread = row)
constexpr int BK = 64;        // columns per chunk (128-byte bf16 rows)

extern __shared__ __align__(128) uint8_t dsm[];

struct DenseParams {
  const uint32_t* gtab;  // byte-field entry table (matvec variant 1)
  int H;
  const qmoe_matrix* mats;
  int E, pass, rows, cols;
  const int32_t* count;  // tokens per expert
  const int32_t* order;  // expert-major token order (qmoe_moe_plan)
  const void* x;
  int x_bf16;
  int64_t ldx;
  void* y;
  int y_mode;
  int64_t ldy;
  int w_off, x_off, plan_off;  // byte offsets in dynamic shared memory
  int dbg;                     // experiment switches (QMOE_DENSE_DBG): 1 skip mma, 2 skip decode
};

__device__ __forceinline__ uint32_t sbase() {
  uint32_t b;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(b) : "l"(dsm));
  return b;
}

__device__ __forceinline__ void sts_u16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v));
}
__device__ __forceinline__ void sts_zero16(uint32_t addr) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(addr), "r"(0u));
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint16_t x_bf16_bits(const void* x, int bf16, int64_t i) {
  if (bf16) return __ldg(reinterpret_cast<const unsigned short*>(x) + i);
  return (uint16_t)(__float_as_uint(__ldg(reinterpret_cast<const float*>(x) + i)) >> 16);  // x is bf16-valued
}

// ------------------------------------------------------------------ tcgen05 variant
// Same decode; the MMA runs on the 5th-generation tensor cores: one elected
// thread issues tcgen05.mma.cta_group::1.kind::f16 (M = 128 rows, N = BN
// tokens, K = 16) from shared-memory descriptors over the SW128 K-major tiles
// (the decode's XOR swizzle IS the canonical 128-byte swizzle), accumulating
// in TMEM (4 row blocks x BN fp32 columns); tcgen05.commit signals an
// mbarrier before the tiles are overwritten. Warp w's TMEM lane quarter holds
// exactly the 32 rows its lanes decoded, read back with tcgen05.ld.32x32b.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // start >> 4 [0,14) | LBO (unused for swizzled K-major) = 1 [16,30) |
  // SBO = 1024 B between 8-row groups [32,46) | version 1 [46,48) | SWIZZLE_128B = 2 [61,64)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int BN>
__device__ __forceinline__ uint32_t idesc_bf16_f32() {
  // c F32 [4,6) | a BF16 [7,10) | b BF16 [10,13) | K-major A, B | N >> 3 [17,23) | M >> 4 [24,29)
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(mb), "r"(parity)
                 : "memory");
}

template <int BN>
__global__ void __launch_bounds__(DTHREADS, 1) dense_tc_kernel(DenseParams P) {
  __shared__ __align__(8) uint64_t tab_bar, mma_bar;
  __shared__ int s_total;
  __shared__ uint32_t s_tmem;
  __shared__ int s_tok[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t base = sbase();
  const uint32_t tab_s = base;
  // operand tiles 1024-byte aligned in the shared window (SW128 atoms)
  const uint32_t w_s = (base + P.w_off + 1023u) & ~1023u, x_s = w_s + (uint32_t)BM * 128u;
  int* start = reinterpret_cast<int*>(dsm + P.plan_off);
  int* ipre = start + P.E + 1;
  const int E = P.E;
  const int nrb = (P.rows + BM - 1) / BM;
  constexpr uint32_t TMEM_COLS = 4 * BN;  // 4 row blocks x BN fp32 columns (128 or 256)
  const uint32_t tb_mb = (uint32_t)__cvta_generic_to_shared(&tab_bar);
  const uint32_t mma_mb = (uint32_t)__cvta_generic_to_shared(&mma_bar);
  if (warp == 0) {  // TMEM accumulators (warp-wide alloc)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tb_mb));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mma_mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)P.H * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tb_mb), "r"(bytes) : "memory");
    for (uint32_t o = 0; o < bytes; o += 32768u)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(tab_s + o),
          "l"(reinterpret_cast<const char*>(P.gtab) + o), "r"(min(32768u, bytes - o)), "r"(tb_mb)
          : "memory");
    int a = 0, it = 0;
    for (int e = 0; e < E; ++e) {
      const int c = __ldg(P.count + e);
      start[e] = a;
      ipre[e] = it;
      a += c;
      it += nrb * ((c + BN - 1) / BN);
    }
    start[E] = a;
    ipre[E] = it;
    s_total = it;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  mbar_wait(tb_mb, 0);
  const uint32_t tmem = s_tmem;
  const int total = s_total;
  const uint32_t H = (uint32_t)P.H;
  const uint32_t rowb = w_s + (uint32_t)tid * 128u;
  const uint32_t rx = (uint32_t)(tid & 7) << 4;
  const uint32_t idesc = idesc_bf16_f32<BN>();
  uint32_t mma_phase = 0;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    int lo = 0, hi = E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ipre[mid] <= item) lo = mid;
      else hi = mid - 1;
    }
    const int e = lo, local = item - ipre[e];
    const int rb = local % nrb, tb = local / nrb;
    const int cnt = start[e + 1] - start[e];
    const int nt = min(BN, cnt - tb * BN);
    const int tok0 = start[e] + tb * BN;
    const qmoe_matrix& M = P.mats[2 * e + P.pass];
    const int r = rb * BM + tid;
    const bool valid = r < P.rows;
    int p = 0, pend = 0, col = 0;
    uint32_t wlo = 0, whi = 0;
    if (valid) {
      p = __ldg(M.row_off + r);
      pend = __ldg(M.row_off + r + 1);
      const uint32_t mm = __ldg(M.row_minmax + r);
      wlo = mm & 0xFFFFu;
      whi = mm >> 16;
    }
    if (tid < BN) s_tok[tid] = tid < nt ? __ldg(P.order + tok0 + tid) : 0;
    __syncthreads();
    constexpr int XPT = BN * BK / DTHREADS;
    uint16_t xr[XPT];
    auto load_x_chunk = [&](int k0) {
#pragma unroll
      for (int u = 0; u < XPT; ++u) {
        const int i = tid + u * DTHREADS, n = i / BK, k = i % BK;
        xr[u] = (n < nt && k0 + k < P.cols) ? x_bf16_bits(P.x, P.x_bf16, (int64_t)s_tok[n] * P.ldx + k0 + k)
                                            : (uint16_t)0;
      }
    };
    load_x_chunk(0);
    // codeword groups: the current group's 8 entries stay looked up across
    // chunks; the next group is prefetched
    const uint16_t* cwp = M.cw;
    const int glast = valid && pend > 0 ? (pend - 1) >> 3 : 0;
    int gcur = -1;
    uint4 gn = make_uint4(0u, 0u, 0u, 0u);
    uint32_t ent[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) ent[u] = 0x007F7F7Fu;
    if (valid && p < pend)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(gn.x), "=r"(gn.y), "=r"(gn.z), "=r"(gn.w)
                   : "l"(cwp + (size_t)(p >> 3) * 8));
    int chunk = 0;
    for (int k0 = 0; k0 < P.cols; k0 += BK, ++chunk) {
      const int k1 = k0 + BK;
      if (chunk > 0) {  // previous chunk's MMAs must be done reading the W / X tiles
        mbar_wait(mma_mb, mma_phase);
        mma_phase ^= 1u;
      }
      const uint32_t xb = x_s + (uint32_t)(chunk & 1) * (BN * 128u);
#pragma unroll
      for (int u = 0; u < XPT; ++u) {
        const int i = tid + u * DTHREADS, n = i / BK, k = i % BK;
        sts_u16(xb + (uint32_t)n * 128u + (((uint32_t)k * 2u) ^ ((uint32_t)(n & 7) << 4)), xr[u]);
      }
      if (k1 < P.cols) load_x_chunk(k1);
#pragma unroll
      for (int c16 = 0; c16 < 8; ++c16) sts_zero16(rowb + 16u * (uint32_t)((c16 + lane) & 7));
      bool go = valid && p < pend && col < k1 && !(P.dbg & 2);
      while (go) {
        const int grp = p >> 3;
        if (grp != gcur) {  // new group: take the prefetched words, look all 8 up, prefetch the next
          const uint4 g = gn;
          gcur = grp;
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(gn.x), "=r"(gn.y), "=r"(gn.z), "=r"(gn.w)
                       : "l"(cwp + (size_t)min(grp + 1, glast) * 8));
          const uint32_t w4[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint32_t c = (u & 1) ? (w4[u >> 1] >> 16) : (w4[u >> 1] & 0xFFFFu);
            ent[u] = c < H ? lds_u32(tab_s + 4 * c) : __ldg(P.gtab + c);
          }
        }
        // walk the group's codewords from p: only the column add is in the chain
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = grp * 8 + u;
          if (go && q >= p) {
            if (q >= pend || col >= k1) {
              go = false;
            } else {
              const uint32_t en = ent[u];
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                const uint32_t f = __byte_perm(en, 0u, 0x4440u + j);
                const int vk = col + (int)(f >> 2) - k0;  // column inside the chunk (f = 0x7F: unused slot)
                if (f != 0x7Fu && (unsigned)vk < (unsigned)BK)
                  sts_u16(rowb + (((uint32_t)vk * 2u) ^ rx), ((en >> (24 + j)) & 1u) ? whi : wlo);
              }
              const int n2 = (int)(en >> 28) * 2;
              if (col + n2 > k1) {
                go = false;  // straddles the chunk end: revisit next chunk
              } else {
                col += n2;
                p = q + 1;
              }
            }
          }
        }
        go = go && p < pend && col < k1;
      }
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0 && (P.dbg & 1)) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mma_mb) : "memory");
      } else if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int mb = 0; mb < BM / 128; ++mb) {
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks) {
            const uint64_t da = sw128_desc(w_s + (uint32_t)mb * 128u * 128u + (uint32_t)ks * 32u);
            const uint64_t db = sw128_desc(xb + (uint32_t)ks * 32u);
            const uint32_t acc = (chunk > 0 || ks > 0) ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
                    tmem + (uint32_t)mb * BN),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mma_mb)
                     : "memory");
      }
    }
    mbar_wait(mma_mb, mma_phase);  // last chunk's MMAs: accumulators final
    mma_phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- epilogue: warp w reads TMEM lanes 32(w%4).. = rows 32w.. of the item, columns of block w/4
    {
      uint32_t v[BN];
      const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * BN;
      if (BN == 64) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,"
            "%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31]), "=r"(v[32 % BN]), "=r"(v[33 % BN]), "=r"(v[34 % BN]),
              "=r"(v[35 % BN]), "=r"(v[36 % BN]), "=r"(v[37 % BN]), "=r"(v[38 % BN]), "=r"(v[39 % BN]),
              "=r"(v[40 % BN]), "=r"(v[41 % BN]), "=r"(v[42 % BN]), "=r"(v[43 % BN]), "=r"(v[44 % BN]),
              "=r"(v[45 % BN]), "=r"(v[46 % BN]), "=r"(v[47 % BN]), "=r"(v[48 % BN]), "=r"(v[49 % BN]),
              "=r"(v[50 % BN]), "=r"(v[51 % BN]), "=r"(v[52 % BN]), "=r"(v[53 % BN]), "=r"(v[54 % BN]),
              "=r"(v[55 % BN]), "=r"(v[56 % BN]), "=r"(v[57 % BN]), "=r"(v[58 % BN]), "=r"(v[59 % BN]),
              "=r"(v[60 % BN]), "=r"(v[61 % BN]), "=r"(v[62 % BN]), "=r"(v[63 % BN])
            : "r"(ta));
      } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (valid) {
#pragma unroll
        for (int n = 0; n < BN; ++n) {
          if (n >= nt) break;
          const int64_t t = s_tok[n];
          const float vv = bf16_round_dev(__uint_as_float(v[n]));
          if (P.y_mode == QMOE_Y_RELU_BF16) {
            reinterpret_cast<uint16_t*>(P.y)[t * P.ldy + r] = (uint16_t)(__float_as_uint(fmaxf(vv, 0.f)) >> 16);
          } else if (P.y_mode == QMOE_Y_STORE_F32) {
            reinterpret_cast<float*>(P.y)[t * P.ldy + r] = vv + 0.f;
          } else {
            float* yp = reinterpret_cast<float*>(P.y) + t * P.ldy + r;
            *yp = *yp + vv;
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM read before the next item's first MMA; token ids reused
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
}

bool al16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

}  // namespace

extern "C" {

int qmoe_dense_moe_pass(qmoe_dict_t d, const uint32_t* d_table, const qmoe_matrix* d_mats, int32_t E, int32_t pass,
                        const int32_t* d_expert_count, const int32_t* d_order, int32_t rows, int32_t cols,
                        const void* d_x, int x_dtype, int64_t ldx, void* d_y, int y_mode, int64_t ldy,
                        int32_t tokens_per_block, int32_t hot_entries, void* stream) {
  if (!d || !d->d_stab || !d_mats || E < 1 || (pass != 0 && pass != 1) || !d_expert_count || !d_order || rows < 0 ||
      cols < 0 || cols % 2 || !d_x || !d_y || (x_dtype != QMOE_X_F32 && x_dtype != QMOE_X_BF16) ||
      (y_mode != QMOE_Y_ACCUM_F32 && y_mode != QMOE_Y_RELU_BF16 && y_mode != QMOE_Y_STORE_F32) ||
      (tokens_per_block != 32 && tokens_per_block != 64))
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (!d->sparse_ok) return qmoe::fail(QMOE_EUNSUPPORTED, "the dense pass needs a <=3-non-zero dictionary");
  if (rows == 0 || cols == 0) return QMOE_OK;
  DenseParams P{};
  P.gtab = (d_table ? d_table : d->d_mtab) + qmoe::MT_STRIDE;
  P.mats = d_mats;
  P.E = E;
  P.pass = pass;
  P.rows = rows;
  P.cols = cols;
  P.count = d_expert_count;
  P.order = d_order;
  P.x = d_x;
  P.x_bf16 = x_dtype == QMOE_X_BF16;
  P.ldx = ldx;
  P.y = d_y;
  P.y_mode = y_mode;
  P.ldy = ldy;
  const int BN = tokens_per_block;
  P.dbg = getenv("QMOE_DENSE_DBG") ? atoi(getenv("QMOE_DENSE_DBG")) : 0;
  const size_t wbytes = (size_t)BM * 128 + 1024, xbytes = (size_t)2 * BN * 128;  // + 1 KB: SW128 alignment
  const size_t plan = ((size_t)(2 * E + 2) * 4 + 127) & ~(size_t)127;
  const size_t static_smem = 1024;
  if (wbytes + xbytes + plan + static_smem + 4096 > (size_t)d->max_smem_optin)
    return qmoe::fail(QMOE_EUNSUPPORTED, "too many experts for the dense pass");
  int H = (int)((d->max_smem_optin - wbytes - xbytes - plan - static_smem) / 4);
  H = std::min(H, hot_entries > 0 ? hot_entries : QMOE_DICT_SIZE) & ~255;
  H = std::max(H, 256);
  P.H = H;
  P.w_off = H * 4;
  P.x_off = P.w_off + (int)wbytes;
  P.plan_off = P.x_off + (int)xbytes;
  const size_t smem = (size_t)P.plan_off + plan;
  const int grid = d->num_sms;
  if (BN == 64) {
    CK(cudaFuncSetAttribute(dense_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    dense_tc_kernel<64><<<grid, DTHREADS, smem, S(stream)>>>(P);
  } else {
    CK(cudaFuncSetAttribute(dense_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    dense_tc_kernel<32><<<grid, DTHREADS, smem, S(stream)>>>(P);
  }
  CK(cudaGetLastError(), "dense_moe_kernel launch");
  (void)al16;
  return QMOE_OK;
}

}  // extern "C"
