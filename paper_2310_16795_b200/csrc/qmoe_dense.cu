// Batched-token decode-then-MMA MoE pass (BASELINE
// configs[2]: Switch-large-128 with many tokens per expert).
//
// With t tokens per expert the streaming matvec re-decodes each expert matrix
// ceil(t / 2) times; here every expert row block is decoded ONCE per step into
// dense bf16 tiles in shared memory and multiplied on the tensor cores with
// all of the expert's tokens (up to 64 per block).
//
//   work item   (expert e, 128-row block, token block of <= BN tokens); the
//               persistent grid strides over the items; every CTA derives the
//               item list from the dispatcher's expert counts (qmoe_moe_plan).
//   decode      thread = row: it walks its row's codewords once, in order,
//               through 64-column chunks; each codeword's <= 3 non-zero bf16
//               levels go into a zero-filled tile whose 16-byte chunks are
//               XOR-swizzled by row (the canonical SW128 K-major UMMA layout);
//               a codeword straddling a chunk end writes its tail into the
//               next tile of a two-tile ring.
//   mma         one thread issues tcgen05.mma (M 128, N = the item's tokens
//               rounded up to 16, K 16) from shared-memory descriptors into a
//               TMEM accumulator, tcgen05.commit on the ring slot's mbarrier;
//               the token tile (bf16) arrives by cp.async one chunk ahead.
//   epilogue    per (row, token): bf16 RNE once (codec.py:243), y mode as the
//               streaming kernel (relu -> bf16 hidden, or f32 store / add).
//
// Numerics: bf16 x bf16 products are exact in fp32; the accumulation order
// differs from the reference's sgemv (tolerance-level parity, as the
// streaming kernel).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <string>

#include "qmoe_device.cuh"

using namespace qmoe_dev;

namespace {

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
  int w_off, plan_off;  // byte offsets in dynamic shared memory
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

// ------------------------------------------------------------------ tcgen05 helpers
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  // start >> 4 [0,14) | LBO 1 (unused, swizzled K-major) [16,30) | SBO 1024 B [32,46) |
  // version 1 [46,48) | SWIZZLE_128B = 2 [61,64)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int BN>
__device__ __forceinline__ uint32_t idesc_bf16_f32() {
  // c F32 [4,6) | a BF16 [7,10) | b BF16 [10,13) | K-major A, B | N >> 3 [17,23) | M = 128: 8 [24,29)
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | (8u << 24);
}

__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(mb), "r"(parity)
                 : "memory");
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint4 ld_group_nc(const uint16_t* cw, int g) {
  // 8 codewords (16-byte aligned group g of the matrix's stream), read once
  uint4 a;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
               : "l"(cw + (size_t)g * 8));
  return a;
}

__device__ __forceinline__ uint32_t lookup_pred(uint32_t cw, uint32_t tab_s, uint32_t H, const uint32_t* gtab) {
  // entry of codeword cw: hot table in shared memory, else global — both
  // loads predicated (no divergent branch: a warp's misses do not serialise)
  uint32_t v;
  asm volatile(
      "{ .reg .pred p; setp.lt.u32 p, %1, %2;\n\t"
      "@p ld.shared.u32 %0, [%3];\n\t"
      "@!p ld.global.nc.u32 %0, [%4]; }"
      : "=r"(v)
      : "r"(cw), "r"(H), "r"(tab_s + 4u * cw), "l"(gtab + cw));
  return v;
}

__device__ __forceinline__ uint32_t group_cw(const uint4& q, uint32_t u) {
  const uint32_t w = (u & 4u) ? ((u & 2u) ? q.w : q.z) : ((u & 2u) ? q.y : q.x);
  return (u & 1u) ? (w >> 16) : (w & 0xFFFFu);
}

// ------------------------------------------------------------------ decode-once kernel
// Item = (expert e, 128-row block, <= BN-token block); thread = row; 64-column
// chunks through a ring of two W tiles (and two token tiles), every codeword
// decoded exactly ONCE per item:
//   codewords   a thread walks its row's codewords in order; chunk k takes
//               the codewords that START before its end column. A codeword
//               spans <= 30 columns, so its values land in tile k or k + 1
//               (zero-filled before chunk k's decode) — no revisits.
//   entries     looked up a group (8 codewords) at a time one refill ahead
//               (registers), then staged in a per-thread ring of 16 entries in
//               shared memory ([slot][thread]: conflict-free); refills happen
//               at a warp-uniform point, not inside the divergent per-codeword
//               loop; the loop itself is branch-free (predicated stores).
//   mma         one thread issues 4 tcgen05.mma (M 128, N = tokens rounded up
//               to 16, K 16) per chunk and commits to the chunk's ring-slot
//               mbarrier; slot k + 1 is rewritten only after MMA(k - 1).
constexpr int DQ_NR = 2, DQ_CTAS = 3, DQ_GE = 16;  // ring slots, CTAs per SM, staged entries per thread

template <int BN>
__global__ void __launch_bounds__(128, DQ_CTAS) dense_dq_kernel(DenseParams P) {
  constexpr int NR = DQ_NR, GE = DQ_GE;
  constexpr uint32_t WT = 128u * 128u;  // W tile: 128 rows x 64 bf16 columns (SW128)
  constexpr uint32_t XT = BN * 128u;    // token tile: BN rows x 64 bf16 columns
  constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  static_assert(NR == 2 && WT == 0x4000u, "column cursor below assumes slot = chunk & 1, tiles 16 KB apart");
  constexpr int XP = BN * 8;              // 16-byte x pieces per chunk
  constexpr int XV = (XP + 127) / 128;    // ... per thread
  __shared__ __align__(8) uint64_t tab_bar, mma_bar[NR];
  __shared__ int s_total;
  __shared__ uint32_t s_tmem;
  __shared__ int s_tok[BN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t base = sbase();
  const uint32_t tab_s = base;
  const uint32_t w_s = (base + P.w_off + 1023u) & ~1023u;
  const uint32_t x_s = w_s + NR * WT;
  const uint32_t ge_s = x_s + NR * XT + 4u * (uint32_t)tid;  // entry ring: slot j at ge_s + 512 j
  int* start = reinterpret_cast<int*>(dsm + P.plan_off);
  int* ipre = start + P.E + 1;
  const int E = P.E;
  const int nrb = (P.rows + 127) / 128;
  const int nk = (P.cols + 63) / 64;
  const uint32_t tb_mb = (uint32_t)__cvta_generic_to_shared(&tab_bar);
  const uint32_t mma_mb0 = (uint32_t)__cvta_generic_to_shared(&mma_bar[0]);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tb_mb));
    for (int i = 0; i < NR; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mma_mb0 + 8u * i));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)P.H * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tb_mb), "r"(bytes) : "memory");
    for (uint32_t o = 0; o < bytes; o += 32768u)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(tab_s + o),
          "l"(reinterpret_cast<const char*>(P.gtab) + o), "r"(min(32768u, bytes - o)), "r"(tb_mb)
          : "memory");
  }
  if (warp == 2) {  // item prefix over experts: warp scan of per-expert item counts
    int carry_t = 0, carry_i = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int c = e < E ? __ldg(P.count + e) : 0;
      const int ni = nrb * ((c + BN - 1) / BN);
      int it = c, ii = ni;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int a = __shfl_up_sync(FULL_MASK, it, d), b = __shfl_up_sync(FULL_MASK, ii, d);
        if (lane >= d) {
          it += a;
          ii += b;
        }
      }
      if (e < E) {
        start[e] = carry_t + it - c;
        ipre[e] = carry_i + ii - ni;
      }
      carry_t += __shfl_sync(FULL_MASK, it, 31);
      carry_i += __shfl_sync(FULL_MASK, ii, 31);
    }
    if (lane == 0) {
      start[E] = carry_t;
      ipre[E] = carry_i;
      s_total = carry_i;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  mbar_wait(tb_mb, 0);
  const uint32_t tmem = s_tmem;
  const int total = s_total;
  const uint32_t H = (uint32_t)P.H;
  const uint32_t rx = (uint32_t)(tid & 7) << 4;  // SW128 16-byte chunk swizzle of my row
  const uint32_t wrow = w_s + (uint32_t)tid * 128u;
  const uint32_t idesc_n0 = idesc_bf16_f32<BN>() & ~(0x3Fu << 17);  // N set per item
  uint32_t mph = 0;  // phase parity of mma_bar[i] in bit i
  auto mma_wait = [&](int slot) {
    mbar_wait(mma_mb0 + 8u * slot, (mph >> slot) & 1u);
    mph ^= 1u << slot;
  };
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
    const uint16_t* cwp = M.cw;
    const int r = rb * 128 + tid;
    int s = 0, n = 0;
    uint32_t wlo = 0, whi = 0;
    if (r < P.rows) {
      s = __ldg(M.row_off + r);
      n = __ldg(M.row_off + r + 1) - s;
      const uint32_t mm = __ldg(M.row_minmax + r);
      wlo = mm & 0xFFFFu;
      whi = mm >> 16;
    }
    if (tid < BN) s_tok[tid] = tid < nt ? __ldg(P.order + tok0 + tid) : 0;
    // codeword cursor, indices relative to my row's first group g0: next
    // codeword i, end iend; entries of [staged - 16, staged) in the ring,
    // entries of group staged / 8 in flight (pe), raw group staged / 8 + 1 in q
    const int g0 = s >> 3, glast = n > 0 ? (s + n - 1) >> 3 : g0;
    int i = s & 7;
    const int iend = i + n;
    // column cursor of codeword i: chunk index << 14 | 0x3F80 (carry bridge)
    // | 2 * (column % 64). Adding a value's byte offset (< 128) carries across
    // the bridge into bit 14 when it leaves the chunk, so (v & 0x407F) is its
    // offset from the ring base: tile (chunk & 1) at 16 KB, row byte in 0..127
    uint32_t colb = 0x3F80u;
    int staged = GE;
    uint32_t pe[8];
    uint4 q;
    {
      const uint4 q0 = ld_group_nc(cwp, g0), q1 = ld_group_nc(cwp, min(g0 + 1, glast));
      const uint4 q2 = ld_group_nc(cwp, min(g0 + 2, glast));
      q = ld_group_nc(cwp, min(g0 + 3, glast));
      uint32_t e0[8], e1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        e0[u] = lookup_pred(group_cw(q0, (uint32_t)u), tab_s, H, P.gtab);
        e1[u] = lookup_pred(group_cw(q1, (uint32_t)u), tab_s, H, P.gtab);
        if (GE == 16) pe[u] = lookup_pred(group_cw(q2, (uint32_t)u), tab_s, H, P.gtab);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ge_s + 512u * u), "r"(e0[u]));
        if (GE == 16) asm volatile("st.shared.u32 [%0], %1;" ::"r"(ge_s + 512u * (u + 8)), "r"(e1[u]));
        else pe[u] = e1[u];
      }
      if (GE == 8) q = q2;
    }
    __syncthreads();  // s_tok
    // token tiles by cp.async (16-byte pieces, zero-filled past the row end
    // and for absent tokens; x is bf16 with ldx % 8 == 0), one commit group
    // per chunk, waited on just before the chunk's MMA
    // MMA N per item: the item's tokens rounded up to 16 (M = 128 needs
    // N % 16 == 0); token-tile rows past it are neither loaded nor read
    const int nmma = (nt + 15) & ~15;
    const uint32_t idesc = idesc_n0 | ((uint32_t)(nmma >> 3) << 17);
    // my pieces' token rows (fixed for the item): x row pointer, or null
    const uint16_t* xrow[XV];
#pragma unroll
    for (int v = 0; v < XV; ++v) {
      const int nn = (tid + v * 128) >> 3;
      xrow[v] = nn < nt ? reinterpret_cast<const uint16_t*>(P.x) + (int64_t)s_tok[nn] * P.ldx : nullptr;
    }
    auto issue_x = [&](int k, int slot) {
      if (k < nk) {
        const int colb0 = k * 64 + (tid & 7) * 8;  // my pieces' first column (c8 = tid & 7 for every v)
        const int nb = 2 * max(0, min(8, P.cols - colb0));
#pragma unroll
        for (int v = 0; v < XV; ++v) {
          const int nn = (tid + v * 128) >> 3;
          const uint32_t dst = x_s + (uint32_t)slot * XT + (uint32_t)nn * 128u + ((uint32_t)((tid & 7) ^ (nn & 7)) << 4);
          if (nn < nmma)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                         "l"(xrow[v] ? xrow[v] + colb0 : reinterpret_cast<const uint16_t*>(P.x)), "r"(xrow[v] ? nb : 0)
                         : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue_x(0, 0);
#pragma unroll
    for (int c16 = 0; c16 < 8; ++c16) sts_zero16(wrow + 16u * (uint32_t)((c16 + lane) & 7));  // tile 0
    int sc = 0;  // ring slot of chunk k
    for (int k = 0; k < nk; ++k) {
      const int sn = sc == NR - 1 ? 0 : sc + 1;
      if (k >= NR - 1) mma_wait(sn);  // MMA(k + 1 - NR) read tiles sn
#pragma unroll
      for (int c16 = 0; c16 < 8; ++c16) sts_zero16(wrow + (uint32_t)sn * WT + 16u * (uint32_t)((c16 + lane) & 7));
      issue_x(k + 1, sn);
      const uint32_t kendb = (uint32_t)(k + 1) << 14;
      for (;;) {
        // warp-uniform refill: the older staged group consumed -> stage the
        // group in flight, look up the next, load the one after
        if (i >= staged - GE + 8 && staged < iend) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(ge_s + 512u * (uint32_t)((staged + u) & (GE - 1))), "r"(pe[u]));
          staged += 8;
#pragma unroll
          for (int u = 0; u < 8; ++u) pe[u] = lookup_pred(group_cw(q, (uint32_t)u), tab_s, H, P.gtab);
          q = ld_group_nc(cwp, min(g0 + (staged >> 3) + 1, glast));
        }
        const int lim = min(staged, iend);
        uint32_t en_n = lds_u32(ge_s + 512u * (uint32_t)(i & (GE - 1)));
        while (i < lim && colb < kendb) {
          const uint32_t en = en_n;  // entry i, loaded an iteration ahead (i + 1 may be stale: reloaded above)
          en_n = lds_u32(ge_s + 512u * (uint32_t)((i + 1) & (GE - 1)));
#pragma unroll
          for (int j = 0; j < 3; ++j) {  // branch-free: the store is predicated on the slot being used
            const uint32_t f = __byte_perm(en, 0u, 0x4440u + j);
            uint32_t a;  // wrow + ((v & 0x407F) ^ rx), the mask and swizzle in one lop3
            asm("lop3.b32 %0, %1, 0x407F, %2, 0x6A;" : "=r"(a) : "r"(colb + (f >> 1)), "r"(rx));
            a += wrow;
            const uint32_t v = ((en >> (24 + j)) & 1u) ? whi : wlo;
            asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 127; @p st.shared.u16 [%0], %1; }" ::"r"(a),
                         "h"((unsigned short)v), "r"(f));
          }
          colb = (colb + (en >> 28) * 4u) | 0x3F80u;
          ++i;
        }
        if (__all_sync(FULL_MASK, i >= iend || colb >= kendb)) break;
      }
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // chunk k's token tile
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t da = sw128_desc(w_s + (uint32_t)sc * WT + (uint32_t)ks * 32u);
          const uint64_t db = sw128_desc(x_s + (uint32_t)sc * XT + (uint32_t)ks * 32u);
          const uint32_t accf = (k > 0 || ks > 0) ? 1u : 0u;
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
                  tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(accf));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         mma_mb0 + 8u * sc)
                     : "memory");
      }
      sc = sn;
    }
    // the last two chunks' MMAs (earlier ones were awaited in the loop)
    for (int kk = max(0, nk - NR + 1); kk < nk; ++kk) mma_wait(kk % NR);
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // the (empty) group past the last chunk
    asm volatile("tcgen05.fence::after_thread_sync;");
    {  // epilogue: warp w reads TMEM lane quarter w (rows), 32 tokens per load
      const int row = rb * 128 + 32 * warp + lane;
#pragma unroll
      for (int half = 0; half < (BN + 31) / 32; ++half) {
        if (half * 32 >= nt) break;
        uint32_t v[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)half * 32u;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < P.rows) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int nn = half * 32 + j;
            if (nn >= nt) break;
            const int64_t t = s_tok[nn];
            const float vv = bf16_round_dev(__uint_as_float(v[j]));
            if (P.y_mode == QMOE_Y_RELU_BF16) {
              reinterpret_cast<uint16_t*>(P.y)[t * P.ldy + row] = (uint16_t)(__float_as_uint(fmaxf(vv, 0.f)) >> 16);
            } else if (P.y_mode == QMOE_Y_STORE_F32) {
              reinterpret_cast<float*>(P.y)[t * P.ldy + row] = vv + 0.f;
            } else {
              float* yp = reinterpret_cast<float*>(P.y) + t * P.ldy + row;
              *yp = *yp + vv;
            }
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
  if (!P.x_bf16 || ldx % 8 != 0 || (reinterpret_cast<uintptr_t>(d_x) & 15) != 0)
    return qmoe::fail(QMOE_EINVAL, "the dense pass needs bf16 x, ldx % 8 == 0 and a 16-byte aligned base");
  {  // 3 CTAs of 128 threads per SM (measured best of 2-4 CTAs x 2-3 ring
     // slots x 8/16 staged entries); the hot table gets the rest of shared memory
    constexpr int DQB = DQ_CTAS, DQR = DQ_NR, DGE = DQ_GE;
    const size_t ring = 1024 + DQR * (size_t)128 * 128 + DQR * (size_t)BN * 128 + DGE * 128 * 4;
    const size_t plan = ((size_t)(2 * E + 2) * 4 + 127) & ~(size_t)127;
    const size_t per_cta = (size_t)d->max_smem_optin / DQB - 1024 - 1024;  // minus static shared memory
    if (ring + plan + 4096 > per_cta) return qmoe::fail(QMOE_EUNSUPPORTED, "too many experts for the dense pass");
    int H = (int)((per_cta - ring - plan) / 4);
    H = std::min(H, hot_entries > 0 ? hot_entries : QMOE_DICT_SIZE) & ~255;
    P.H = std::max(H, 256);
    P.w_off = P.H * 4;
    P.plan_off = P.w_off + (int)ring;
    const size_t smem = (size_t)P.plan_off + plan;
    const int grid = DQB * d->num_sms;
    if (BN == 64) {
      CK(cudaFuncSetAttribute(dense_dq_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
         "attr");
      dense_dq_kernel<64><<<grid, 128, smem, S(stream)>>>(P);
    } else {
      CK(cudaFuncSetAttribute(dense_dq_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
         "attr");
      dense_dq_kernel<32><<<grid, 128, smem, S(stream)>>>(P);
    }
    CK(cudaGetLastError(), "dense_dq_kernel launch");
    return QMOE_OK;
  }
}

}  // extern "C"
