// Fused dictionary-decode + matvec (codec.py:196-244 semantics) for sm_100a.
//
// stream_matvec_kernel — the product path for dictionaries whose entries hold
// <= 3 non-zero values (the default p0 = 0.885 dictionary). Persistent, one
// CTA per SM, warp-specialised:
//   * warp 0 = producer. It keeps the work records of the next units in a
//     shared-memory ring (refilled one 32-record batch ahead from registers)
//     and lane 0 stages, per work unit, the unit's codeword range, row
//     offsets, row scales, row checkpoints and (when the tokens change) the x
//     rows into a STAGES-deep ring of shared-memory slots with cp.async.bulk,
//     completing a `full` mbarrier; a slot is reused once all consumer warps
//     arrived on its `empty` mbarrier.
//   * warps 1..15 = consumers. A unit's rows are dealt out as tasks of
//     32/G rows (shared-memory atomic dispenser). Within a task each lane owns
//     one contiguous SEGMENT of one row (G = 2^lg segments per row; lg = 0:
//     a lane per row) and walks it with a running column offset that starts
//     at the row's checkpoint — no scans, no scratch. Codewords are looked up
//     8 at a time, the next batch issued before the current one is applied
//     (hot prefix of the packed entry table in shared memory, the rest through
//     the read-only path). Per non-zero slot: S += x (every non-zero) and
//     T += x (code-2 non-zeros); a row's result is lmin*S + (lmax-lmin)*T
//     (= lmin*S1 + lmax*S2), reduced over its G lanes, bf16-rounded once
//     (codec.py:243).
//   * the entry table prefix is filled by one bulk copy at kernel start.
// Entry format "matvec" (built in qmoe_host.cpp, esz = bytes per staged x):
//   bits 0-4 len = 2n | bits 5-11, 12-18, 19-25: position * esz of non-zero
//   slot 0..2 | bits 26-28 slot used | bits 29-31 slot is code 2 (row max).
//
// general_matvec_kernel — any dictionary (e.g. p0 = 0.7, up to 6 non-zeros per
// entry): expands the two decode words value by value (dictionary.py:115-120).
#include <algorithm>
#include <climits>

#include "qmoe_device.cuh"

using namespace qmoe_dev;

namespace {

constexpr int NCONS = 15;                  // consumer warps (16 warps total: 4 per SMSP)
constexpr int THREADS = (NCONS + 1) * 32;  // + one producer warp
constexpr int STAGES = 8;
constexpr int CW_CAP = 3072;               // codewords per staged unit
constexpr int ROW_CAP = 128;               // rows per staged unit
constexpr int BATCH = 8;                   // codewords looked up per batch per lane
constexpr uint32_t COLD_ZERO = 65536;      // tables carry zero entries from here
constexpr int NT_STREAM = 2;               // tokens per unit on the streaming path
constexpr int RING = 64;                   // producer record ring

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int ESZ>
struct XType;
template <>
struct XType<4> {
  using T = float;
  static __device__ __forceinline__ float get(float v) { return v; }
};
template <>
struct XType<2> {
  using T = uint16_t;
  static __device__ __forceinline__ float get(uint16_t v) { return __uint_as_float(uint32_t(v) << 16); }
};

// ----------------------------------------------------------------- records
struct Rec {  // == qmoe_work (80 bytes)
  const uint16_t* cw;
  const int32_t* ro;
  const uint32_t* mm;
  const uint16_t* ck;
  int32_t cols, row0, row1, ntok, cw0, cw1, lg, pad;
  int32_t tok[QMOE_NT_MAX];
};
static_assert(sizeof(Rec) == sizeof(qmoe_work), "record layout");

// per-slot staging metadata written by the producer before the full arrive
struct SlotMeta {
  Rec r;
  uint32_t cw_s, ro_s, mm_s, ck_s, x_s;  // byte offsets (from the smem base) of the staged ranges
  int32_t direct;                        // 1: unit exceeds the slot, read global
  int32_t next;                          // task dispenser (smem atomic)
  int32_t pad;
};

struct StreamParams {
  const uint32_t* gtab;       // matvec-format table variant (zero entries from 65536)
  int H;                      // entries staged in shared memory
  const qmoe_work* work;      // explicit work list (or nullptr: implicit single matrix)
  const int32_t* n_work;
  int max_work;
  qmoe_matrix single;         // implicit mode (lane per row, no checkpoints)
  int rows_per_unit;
  int64_t ntok_single;
  int ntu_single;
  const void* x;
  int64_t ldx;
  void* y;
  int y_mode;
  int64_t ldy;
  int32_t* bad;
  int xcap;                   // elements per token slot of an x buffer
  int ntmax;                  // token slots per x buffer
};

__device__ __forceinline__ void make_rec(const StreamParams& P, int u, Rec& R) {
  if (P.work) {
    const uint4* s = reinterpret_cast<const uint4*>(P.work + u);
    uint4* d = reinterpret_cast<uint4*>(&R);
#pragma unroll
    for (int i = 0; i < 5; ++i) d[i] = __ldg(s + i);
  } else {
    const int nblk = (P.single.rows + P.rows_per_unit - 1) / P.rows_per_unit;
    const int chunk = u / nblk, blk = u % nblk;
    R.cw = P.single.cw;
    R.ro = P.single.row_off;
    R.mm = P.single.row_minmax;
    R.ck = nullptr;
    R.cols = P.single.cols;
    R.lg = 0;
    R.pad = 0;
    R.row0 = blk * P.rows_per_unit;
    R.row1 = min(P.single.rows, R.row0 + P.rows_per_unit);
    const int64_t t0 = (int64_t)chunk * P.ntu_single;
    R.ntok = (int)min((int64_t)P.ntu_single, P.ntok_single - t0);
#pragma unroll
    for (int q = 0; q < QMOE_NT_MAX; ++q) R.tok[q] = (int)(t0 + min(q, R.ntok - 1));
    R.cw0 = __ldg(R.ro + R.row0);
    R.cw1 = __ldg(R.ro + R.row1);
  }
}

__device__ __forceinline__ bool same_x(const Rec& a, const Rec& b) {
  bool s = a.cols == b.cols && a.ntok == b.ntok;
#pragma unroll
  for (int q = 0; q < QMOE_NT_MAX; ++q) s = s && (q >= a.ntok || a.tok[q] == b.tok[q]);
  return s;
}

__device__ __forceinline__ uint32_t span(const void* begin, size_t nbytes, uint32_t& delta, uintptr_t& a0) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(begin);
  a0 = a & ~uintptr_t(15);
  delta = (uint32_t)(a - a0);
  return (uint32_t)(((a + nbytes + 15) & ~uintptr_t(15)) - a0);
}

// ----------------------------------------------------------------- consumer
// Look up BATCH codewords of this lane's segment starting at k0 (past the
// segment's end: the zero entry at COLD_ZERO).
__device__ __forceinline__ void lookup_batch(uint32_t (&t)[BATCH], const uint16_t* cw, int cnt, int k0,
                                             const uint32_t* tab, uint32_t H, const uint32_t* __restrict__ gtab) {
#pragma unroll
  for (int u = 0; u < BATCH; ++u) {
    const uint32_t c = (k0 + u < cnt) ? (uint32_t)cw[k0 + u] : COLD_ZERO;
    t[u] = c < H ? tab[c] : __ldg(gtab + c);
  }
}

// Apply BATCH entries at the running column `off` (elements).
template <int NT, int ESZ>
__device__ __forceinline__ void apply_batch(const uint32_t (&t)[BATCH], const typename XType<ESZ>::T* xs, int xslot,
                                            int& off, float (&S)[NT], float (&T)[NT]) {
  using XT = typename XType<ESZ>::T;
#pragma unroll
  for (int u = 0; u < BATCH; ++u) {
    const uint32_t e = t[u];
    const char* xo = reinterpret_cast<const char*>(xs + off);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const bool used = (e >> (26 + j)) & 1u;
      const bool two = (e >> (29 + j)) & 1u;
      const XT* xp = reinterpret_cast<const XT*>(xo + ((e >> (5 + 7 * j)) & 0x7Fu));
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const float v = used ? XType<ESZ>::get(xp[q * xslot]) : 0.f;
        S[q] += v;
        T[q] += two ? v : 0.f;
      }
    }
    off += int(e & 31u);
  }
}

template <int NT, int ESZ>
__device__ __forceinline__ void run_unit(const StreamParams& P, SlotMeta& M, const uint8_t* smem) {
  using XT = typename XType<ESZ>::T;
  const int lane = threadIdx.x & 31;
  // everything the task loop needs, read once
  const int row0 = M.r.row0, nrows = M.r.row1 - M.r.row0, cw0 = M.r.cw0, cols = M.r.cols, ntok = M.r.ntok;
  const int lg = M.r.lg;
  int tok[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) tok[q] = M.r.tok[q];
  const uint16_t* cwp = reinterpret_cast<const uint16_t*>(smem + M.cw_s);
  const int32_t* rop = reinterpret_cast<const int32_t*>(smem + M.ro_s);
  const uint32_t* mmp = reinterpret_cast<const uint32_t*>(smem + M.mm_s);
  const uint16_t* ckp = reinterpret_cast<const uint16_t*>(smem + M.ck_s);
  const XT* xs = reinterpret_cast<const XT*>(smem + M.x_s);
  const uint32_t* tab = reinterpret_cast<const uint32_t*>(smem);
  int32_t* next = &M.next;
  const int G = 1 << lg;
  const int rg = lane >> lg, seg = lane & (G - 1);
  const int ntasks = (nrows + (32 >> lg) - 1) >> (5 - lg);
  const uint32_t H = (uint32_t)P.H;
  const uint32_t* gtab = P.gtab;
  const int xslot = P.xcap;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(next, 1);
    task = __shfl_sync(FULL_MASK, task, 0);
    if (task >= ntasks) break;
    const int i = (task << (5 - lg)) + rg;
    const bool valid = i < nrows;
    int b = 0, cnt = 0, off = 0;
    uint32_t mm = 0;
    if (valid) {
      const int s = rop[i] - cw0;
      const int n = rop[i + 1] - rop[i];
      b = s + ((seg * n) >> lg);
      cnt = s + (((seg + 1) * n) >> lg) - b;
      off = seg ? (int)ckp[i * (G - 1) + seg - 1] : 0;
      mm = mmp[i];
    }
    const int maxc = __reduce_max_sync(FULL_MASK, cnt);
    float S[NT], T[NT];
#pragma unroll
    for (int q = 0; q < NT; ++q) S[q] = T[q] = 0.f;
    const uint16_t* c = cwp + b;
    uint32_t ta[BATCH], tb[BATCH];
    lookup_batch(ta, c, cnt, 0, tab, H, gtab);
    for (int k0 = 0;;) {
      if (k0 + BATCH < maxc) lookup_batch(tb, c, cnt, k0 + BATCH, tab, H, gtab);
      apply_batch<NT, ESZ>(ta, xs, xslot, off, S, T);
      k0 += BATCH;
      if (k0 >= maxc) break;
      if (k0 + BATCH < maxc) lookup_batch(ta, c, cnt, k0 + BATCH, tab, H, gtab);
      apply_batch<NT, ESZ>(tb, xs, xslot, off, S, T);
      k0 += BATCH;
      if (k0 >= maxc) break;
    }
#pragma unroll
    for (int q = 0; q < NT; ++q) {
#pragma unroll
      for (int d = 1; d < 32; d <<= 1)
        if (d < G) {
          S[q] += __shfl_xor_sync(FULL_MASK, S[q], d);
          T[q] += __shfl_xor_sync(FULL_MASK, T[q], d);
        }
    }
    if (!valid || seg != G - 1) continue;  // the last segment's lane ends the row
    const int r = row0 + i;
    if (off != cols) {  // row decodes to the wrong number of values: never written
      if (P.bad) {
        atomicAdd(P.bad, 1);
        atomicMin(P.bad + 1, r);
      }
      continue;
    }
    const float lmin = __uint_as_float(mm << 16), lmax = __uint_as_float(mm & 0xFFFF0000u);
    const float dl = lmax - lmin;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      if (q >= ntok) break;
      const float v = bf16_round_dev(fmaf(lmin, S[q], dl * T[q]));
      if (P.y_mode == QMOE_Y_RELU_BF16) {
        uint16_t* yp = reinterpret_cast<uint16_t*>(P.y) + (int64_t)tok[q] * P.ldy + r;
        *yp = (uint16_t)(__float_as_uint(fmaxf(v, 0.f)) >> 16);
      } else if (P.y_mode == QMOE_Y_STORE_F32) {
        reinterpret_cast<float*>(P.y)[(int64_t)tok[q] * P.ldy + r] = v + 0.f;  // == 0 + v
      } else {
        float* yp = reinterpret_cast<float*>(P.y) + (int64_t)tok[q] * P.ldy + r;
        *yp = *yp + v;
      }
    }
  }
}

// Slow path for units larger than a slot: everything read from global.
template <int ESZ>
__device__ void run_unit_direct(const StreamParams& P, const SlotMeta& M, int cwarp) {
  const Rec& R = M.r;
  const int lane = threadIdx.x & 31;
  for (int i = cwarp; i < R.row1 - R.row0; i += NCONS) {
    const int r = R.row0 + i;
    const int s = __ldg(R.ro + r), e = __ldg(R.ro + r + 1);
    const uint32_t mm = __ldg(R.mm + r);
    const float lmin = __uint_as_float(mm << 16), lmax = __uint_as_float(mm & 0xFFFF0000u);
    float acc0 = 0.f, acc1 = 0.f;
    int base = 0;
    for (int p0 = s; p0 < e; p0 += 32) {
      const uint32_t c = p0 + lane < e ? (uint32_t)__ldg(R.cw + p0 + lane) : COLD_ZERO;
      const uint32_t t = __ldg(P.gtab + c);
      const int len = int(t & 31u);
      int incl = len;
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(FULL_MASK, incl, d);
        if (lane >= d) incl += v;
      }
      const int off = base + incl - len;
      base += __shfl_sync(FULL_MASK, incl, 31);
      for (int j = 0; j < 3; ++j) {
        if (!((t >> (26 + j)) & 1u)) continue;
        const int col = off + int(((t >> (5 + 7 * j)) & 0x7Fu) / ESZ);
        const float w = ((t >> (29 + j)) & 1u) ? lmax : lmin;
        for (int q = 0; q < R.ntok && q < 2; ++q) {
          const int64_t xi = (int64_t)R.tok[q] * P.ldx + col;
          const float xv = ESZ == 2 ? __uint_as_float(uint32_t(__ldg(reinterpret_cast<const uint16_t*>(P.x) + xi)) << 16)
                                    : __ldg(reinterpret_cast<const float*>(P.x) + xi);
          if (q == 0) acc0 = fmaf(w, xv, acc0);
          else acc1 = fmaf(w, xv, acc1);
        }
      }
    }
    acc0 = warp_sum(acc0);
    acc1 = warp_sum(acc1);
    if (lane != 0) continue;
    if (base != R.cols) {
      if (P.bad) {
        atomicAdd(P.bad, 1);
        atomicMin(P.bad + 1, r);
      }
      continue;
    }
    for (int q = 0; q < R.ntok && q < 2; ++q) {
      const float v = bf16_round_dev(q == 0 ? acc0 : acc1);
      if (P.y_mode == QMOE_Y_RELU_BF16)
        reinterpret_cast<uint16_t*>(P.y)[(int64_t)R.tok[q] * P.ldy + r] = (uint16_t)(__float_as_uint(fmaxf(v, 0.f)) >> 16);
      else if (P.y_mode == QMOE_Y_STORE_F32)
        reinterpret_cast<float*>(P.y)[(int64_t)R.tok[q] * P.ldy + r] = v + 0.f;
      else {
        float* yp = reinterpret_cast<float*>(P.y) + (int64_t)R.tok[q] * P.ldy + r;
        *yp = *yp + v;
      }
    }
  }
}

struct Carve {
  uint32_t tab_s, bar_full, bar_empty, bar_tab, cwbuf, robuf, mmbuf, ckbuf, xbuf, xbytes;
  SlotMeta* meta;
  Rec* ring;  // producer's record ring [RING]
};

// Producer warp: keeps the records of the next 32 units in flight in
// registers, the current ones in a shared-memory ring, and stages one unit
// per iteration into the ring of STAGES slots (lane 0 issues the bulk copies).
template <int ESZ>
__device__ __noinline__ void producer(const StreamParams& P, const Carve& C, int u0, int u1) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    mbar_arrive_expect_tx(C.bar_tab, (uint32_t)P.H * 4);
    if (P.H > 0) bulk_g2s(C.tab_s, P.gtab, (uint32_t)P.H * 4, C.bar_tab);
  }
  Rec nxt;
  for (int v = u0 + lane; v < min(u1, u0 + RING); v += 32) {
    Rec r;
    make_rec(P, v, r);
    C.ring[(v - u0) % RING] = r;
  }
  if (u0 + RING + lane < u1) make_rec(P, u0 + RING + lane, nxt);
  __syncwarp();
  int cur_xb = 1;
  int last_x0 = -1, last_x1 = -1;  // last unit that used x buffer 0 / 1
  int consumed = -1;               // highest relative unit known consumed
  for (int u = u0; u < u1; ++u) {
    const int rel = u - u0;
    if (lane == 0) {
      const Rec& R = C.ring[rel % RING];
      const int s = rel % STAGES;
      if (rel >= STAGES) {
        while (consumed < rel - STAGES) {
          ++consumed;
          mbar_wait(C.bar_empty + 8 * (consumed % STAGES), (uint32_t)((consumed / STAGES) & 1));
        }
      }
      SlotMeta& M = C.meta[s];
      const int nrows = R.row1 - R.row0;
      const int ncw = R.cw1 - R.cw0;
      const int nck = (1 << R.lg) - 1;
      M.r = R;
      M.direct = (ncw > CW_CAP || nrows > ROW_CAP || nck > 7) ? 1 : 0;
      M.next = 0;
      const bool reuse = rel > 0 && same_x(C.ring[(rel - 1) % RING], R);
      int xb = cur_xb;
      if (!reuse) {
        xb = cur_xb ^ 1;
        const int v = xb ? last_x1 : last_x0;
        while (v >= 0 && consumed < v) {
          ++consumed;
          mbar_wait(C.bar_empty + 8 * (consumed % STAGES), (uint32_t)((consumed / STAGES) & 1));
        }
      }
      if (xb) last_x1 = rel;
      else last_x0 = rel;
      cur_xb = xb;
      M.x_s = C.xbuf + (uint32_t)xb * C.xbytes - C.tab_s;
      const uint32_t full = C.bar_full + 8 * s;
      const uint32_t cw_dst = C.cwbuf + s * (CW_CAP * 2 + 64);
      const uint32_t ro_dst = C.robuf + s * (ROW_CAP * 4 + 64);
      const uint32_t mm_dst = C.mmbuf + s * (ROW_CAP * 4 + 64);
      const uint32_t ck_dst = C.ckbuf + s * (ROW_CAP * 2 * 7 + 64);
      uintptr_t acw = 0, aro = 0, amm = 0, ack = 0;
      uint32_t bcw = 0, bro = 0, bmm = 0, bck = 0, dcw = 0, dro = 0, dmm = 0, dck = 0, total = 0;
      if (!M.direct) {
        bcw = span(R.cw + R.cw0, (size_t)ncw * 2, dcw, acw);
        bro = span(R.ro + R.row0, (size_t)(nrows + 1) * 4, dro, aro);
        bmm = span(R.mm + R.row0, (size_t)nrows * 4, dmm, amm);
        if (nck) bck = span(R.ck + (size_t)R.row0 * nck, (size_t)nrows * nck * 2, dck, ack);
        total = bcw + bro + bmm + bck;
      }
      const size_t xrow = (size_t)R.cols * ESZ;
      const uint32_t xrow16 = (uint32_t)((xrow + 15) & ~size_t(15));  // x rows are 16-byte aligned
      if (!reuse) total += xrow16 * (uint32_t)R.ntok;
      M.cw_s = cw_dst + dcw - C.tab_s;
      M.ro_s = ro_dst + dro - C.tab_s;
      M.mm_s = mm_dst + dmm - C.tab_s;
      M.ck_s = ck_dst + dck - C.tab_s;
      fence_proxy_async();
      mbar_arrive_expect_tx(full, total);  // releases M.* to the consumers
      if (bcw) bulk_g2s(cw_dst, reinterpret_cast<const void*>(acw), bcw, full);
      if (bro) bulk_g2s(ro_dst, reinterpret_cast<const void*>(aro), bro, full);
      if (bmm) bulk_g2s(mm_dst, reinterpret_cast<const void*>(amm), bmm, full);
      if (bck) bulk_g2s(ck_dst, reinterpret_cast<const void*>(ack), bck, full);
      if (!reuse) {
        for (int q = 0; q < R.ntok; ++q)
          bulk_g2s(C.tab_s + M.x_s + (uint32_t)q * P.xcap * ESZ,
                   reinterpret_cast<const uint8_t*>(P.x) + (int64_t)R.tok[q] * P.ldx * ESZ, xrow16, full);
      }
    }
    // after the last unit of a 32-batch: park the prefetched records in the
    // ring half that just drained and prefetch the next batch
    if ((rel & 31) == 31) {
      __syncwarp();
      const int v = u + 1 + (RING - 32) + lane;
      if (v < u1) C.ring[(v - u0) % RING] = nxt;
      __syncwarp();
      if (v + 32 < u1) make_rec(P, v + 32, nxt);
    }
    __syncwarp();
  }
}

template <int ESZ>
__global__ void __launch_bounds__(THREADS, 1) stream_matvec_kernel(StreamParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  Carve C;
  C.tab_s = saddr(smem);
  uint8_t* p = smem + (size_t)P.H * 4;
  C.bar_full = saddr(p);  // STAGES x 8
  C.bar_empty = C.bar_full + 8 * STAGES;
  C.bar_tab = C.bar_empty + 8 * STAGES;
  p += 128;
  C.meta = reinterpret_cast<SlotMeta*>(p);
  p += ((sizeof(SlotMeta) * STAGES + 127) / 128) * 128;
  C.ring = reinterpret_cast<Rec*>(p);
  p += sizeof(Rec) * RING;
  C.cwbuf = saddr(p);
  p += STAGES * (CW_CAP * 2 + 64);
  C.robuf = saddr(p);
  p += STAGES * (ROW_CAP * 4 + 64);
  C.mmbuf = saddr(p);
  p += STAGES * (ROW_CAP * 4 + 64);
  C.ckbuf = saddr(p);
  p += STAGES * (ROW_CAP * 2 * 7 + 64);
  C.xbuf = saddr(p);  // [2][ntmax][xcap]
  C.xbytes = (uint32_t)P.ntmax * P.xcap * ESZ;

  int n;
  if (P.work) n = min(*P.n_work, P.max_work);
  else {
    const int nblk = (P.single.rows + P.rows_per_unit - 1) / P.rows_per_unit;
    n = nblk * (int)((P.ntok_single + P.ntu_single - 1) / P.ntu_single);
  }
  const int u0 = (int)((int64_t)n * blockIdx.x / gridDim.x);
  const int u1 = (int)((int64_t)n * (blockIdx.x + 1) / gridDim.x);
  if (u0 >= u1) return;  // whole CTA exits before any barrier use

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(C.bar_full + 8 * s, 1);
      mbar_init(C.bar_empty + 8 * s, NCONS);
    }
    mbar_init(C.bar_tab, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    producer<ESZ>(P, C, u0, u1);
  } else {
    const int cwarp = warp - 1;
    mbar_wait(C.bar_tab, 0);
    for (int u = u0; u < u1; ++u) {
      const int rel = u - u0;
      const int s = rel % STAGES;
      mbar_wait(C.bar_full + 8 * s, (uint32_t)((rel / STAGES) & 1));
      SlotMeta& M = C.meta[s];
      if (M.direct) run_unit_direct<ESZ>(P, M, cwarp);
      else if (M.r.ntok == 1) run_unit<1, ESZ>(P, M, smem);
      else run_unit<2, ESZ>(P, M, smem);
      __syncwarp();
      if (lane == 0) mbar_arrive(C.bar_empty + 8 * s);
    }
  }
}

// ----------------------------------------------------------------- general path
// Any dictionary: decode words read through the cache, value-by-value walk.
// Warp per row over a flat work list; exact, not the tuned path.
struct GeneralParams {
  const uint32_t* words;
  const qmoe_work* work;
  const int32_t* n_work;
  int max_work;
  qmoe_matrix single;
  int64_t ntok_single;
  const void* x;
  int x_bf16;
  int64_t ldx;
  void* y;
  int y_mode;
  int64_t ldy;
  int32_t* bad;
};

__global__ void __launch_bounds__(256) general_matvec_kernel(GeneralParams P) {
  const int lane = threadIdx.x & 31;
  const int n = P.work ? min(*P.n_work, P.max_work) : (int)P.ntok_single;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int u = 0; u < n; ++u) {
    const uint16_t* cw;
    const int32_t* ro;
    const uint32_t* mmv;
    int cols, row0, row1, ntok, tok[QMOE_NT_MAX];
    if (P.work) {
      const qmoe_work W = P.work[u];
      cw = W.cw;
      ro = W.row_off;
      mmv = W.row_minmax;
      cols = W.cols;
      row0 = W.row0;
      row1 = W.row1;
      ntok = W.ntok;
      for (int q = 0; q < QMOE_NT_MAX; ++q) tok[q] = W.tok[q];
    } else {
      cw = P.single.cw;
      ro = P.single.row_off;
      mmv = P.single.row_minmax;
      cols = P.single.cols;
      row0 = 0;
      row1 = P.single.rows;
      ntok = 1;
      tok[0] = u;
    }
    for (int r = row0 + w0; r < row1; r += nw) {
      const int s = __ldg(ro + r), e = __ldg(ro + r + 1);
      float acc[QMOE_NT_MAX] = {0, 0, 0, 0};
      const uint32_t mm = __ldg(mmv + r);
      const float lmin = __uint_as_float(mm << 16), lmax = __uint_as_float(mm & 0xFFFF0000u);
      int base = 0;
      for (int p0 = s; p0 < e; p0 += 32) {
        const int i = p0 + lane;
        uint2 w = make_uint2(0u, 0u);
        if (i < e) w = __ldg(reinterpret_cast<const uint2*>(P.words) + __ldg(cw + i));
        const int len = 2 * int(w.x & 15u);
        int incl = len;
        for (int d = 1; d < 32; d <<= 1) {
          const int v = __shfl_up_sync(FULL_MASK, incl, d);
          if (lane >= d) incl += v;
        }
        const int off = base + incl - len;
        base += __shfl_sync(FULL_MASK, incl, 31);
        for (int v = 0; v < len; ++v) {
          const uint32_t code = ((v < 14 ? w.x : w.y) >> (4 + 2 * (v % 14))) & 3u;
          if (!code || off + v >= cols) continue;
          const float lv = code == 1u ? lmin : lmax;
          for (int q = 0; q < ntok; ++q) {
            const int64_t xi = (int64_t)tok[q] * P.ldx + off + v;
            const float xv = P.x_bf16 ? __uint_as_float(uint32_t(__ldg(reinterpret_cast<const uint16_t*>(P.x) + xi)) << 16)
                                      : __ldg(reinterpret_cast<const float*>(P.x) + xi);
            acc[q] = fmaf(lv, xv, acc[q]);
          }
        }
      }
      for (int q = 0; q < QMOE_NT_MAX; ++q) acc[q] = warp_sum(acc[q]);
      if (lane != 0) continue;
      if (base != cols) {
        if (P.bad) {
          atomicAdd(P.bad, 1);
          atomicMin(P.bad + 1, r);
        }
        continue;
      }
      for (int q = 0; q < ntok; ++q) {
        const float v = bf16_round_dev(acc[q]);
        if (P.y_mode == QMOE_Y_RELU_BF16) {
          reinterpret_cast<uint16_t*>(P.y)[(int64_t)tok[q] * P.ldy + r] = (uint16_t)(__float_as_uint(fmaxf(v, 0.f)) >> 16);
        } else if (P.y_mode == QMOE_Y_STORE_F32) {
          reinterpret_cast<float*>(P.y)[(int64_t)tok[q] * P.ldy + r] = v + 0.f;
        } else {
          float* yp = reinterpret_cast<float*>(P.y) + (int64_t)tok[q] * P.ldy + r;
          *yp = *yp + v;
        }
      }
    }
  }
}

// ----------------------------------------------------------------- host side
size_t fixed_smem() {
  return 128 + ((sizeof(SlotMeta) * STAGES + 127) / 128) * 128 + sizeof(Rec) * RING +
         STAGES * (CW_CAP * 2 + 64) + 2 * STAGES * (ROW_CAP * 4 + 64) + STAGES * (ROW_CAP * 2 * 7 + 64);
}

int hot_override() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("QMOE_HOT_ENTRIES");
    v = e ? atoi(e) : -1;
  }
  return v;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int launch_stream(const qmoe_dict* d, StreamParams& P, int esz, int max_cols, int ntmax, int grid, int hot_want,
                  cudaStream_t st) {
  P.ntmax = ntmax;
  P.xcap = ((max_cols + 32 + 15) / 16) * 16;
  const size_t xbytes = 2 * (size_t)ntmax * P.xcap * esz;
  const size_t fixed = fixed_smem() + xbytes;
  if (fixed + 4096 > (size_t)d->max_smem_optin)
    return qmoe::fail(QMOE_EUNSUPPORTED, "cols too large for the shared-memory x staging buffer");
  int H = (int)((d->max_smem_optin - fixed) / 4);
  if (hot_override() >= 0) hot_want = hot_override();
  H = std::min(H, std::min(hot_want, QMOE_DICT_SIZE));
  H &= ~255;
  P.H = H;
  const size_t smem = (size_t)H * 4 + fixed;
  if (esz == 2) {
    CK(cudaFuncSetAttribute(stream_matvec_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    stream_matvec_kernel<2><<<grid, THREADS, smem, st>>>(P);
  } else {
    CK(cudaFuncSetAttribute(stream_matvec_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    stream_matvec_kernel<4><<<grid, THREADS, smem, st>>>(P);
  }
  CK(cudaGetLastError(), "stream_matvec_kernel launch");
  return QMOE_OK;
}

const uint32_t* pick_table(const qmoe_dict* d, const uint32_t* user, int esz) {
  // tables hold both variants back to back: [esz 4 | esz 2], MT_STRIDE entries each
  if (user) return esz == 4 ? user : user + qmoe::MT_STRIDE;
  return esz == 4 ? d->d_mtab : d->d_mtab + qmoe::MT_STRIDE;
}

}  // namespace

extern "C" {

static int fused_common(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, const uint32_t* d_mm,
                        int64_t rows, int64_t cols, const void* d_x, int x_dtype, int64_t ntok, int64_t ldx,
                        float* d_y, int64_t ldy, int32_t* d_bad, void* stream) {
  if (!d || !d->d_stab || rows < 0 || cols < 0 || cols % 2 || ntok < 0 ||
      (x_dtype != QMOE_X_F32 && x_dtype != QMOE_X_BF16))
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  if (rows > INT32_MAX / 2 || cols > INT32_MAX / 2) return qmoe::fail(QMOE_EINVAL, "matrix too large");
  if (rows == 0 || ntok == 0 || cols == 0) return QMOE_OK;
  const int esz = x_dtype == QMOE_X_BF16 ? 2 : 4;
  if (!aligned16(d_cw) || !aligned16(d_row_off) || !aligned16(d_mm) || !aligned16(d_x) || (ldx * esz) % 16)
    return qmoe::fail(QMOE_EINVAL, "device arrays must be 16-byte aligned (and x rows 16-byte strided)");
  if (d->sparse_ok) {
    // rows per unit from a typical ~24 values per codeword (no host sync; a
    // unit that outgrows a slot is read directly from global)
    const double per_row = std::max(1.0, (double)cols / 24.0);
    const int rpu = (int)std::max(1.0, std::min(0.75 * CW_CAP / per_row, (double)ROW_CAP));
    const int ntu = (int)std::min<int64_t>(ntok, NT_STREAM);
    StreamParams P{};
    P.gtab = pick_table(d, nullptr, esz);
    P.work = nullptr;
    P.single = qmoe_matrix{d_cw, d_row_off, d_mm, nullptr, (int32_t)rows, (int32_t)cols, 0, 0};
    P.rows_per_unit = rpu;
    P.ntok_single = ntok;
    P.ntu_single = ntu;
    P.x = d_x;
    P.ldx = ldx;
    P.y = d_y;
    P.y_mode = QMOE_Y_ACCUM_F32;
    P.ldy = ldy;
    P.bad = d_bad;
    const int64_t nblk = (rows + rpu - 1) / rpu;
    const int64_t units = nblk * ((ntok + ntu - 1) / ntu);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, d->num_sms));
    // small launches stage a smaller hot table (the fill is per CTA)
    const int64_t est_cw = rows * cols / 24 + rows;
    const int want = (int)std::min<int64_t>(QMOE_DICT_SIZE, std::max<int64_t>(4096, est_cw / grid * 2));
    return launch_stream(d, P, esz, (int)cols, ntu, grid, want, S(stream));
  }
  GeneralParams G{};
  G.words = d->d_words;
  G.single = qmoe_matrix{d_cw, d_row_off, d_mm, nullptr, (int32_t)rows, (int32_t)cols, 0, 0};
  G.ntok_single = ntok;
  G.x = d_x;
  G.x_bf16 = x_dtype == QMOE_X_BF16;
  G.ldx = ldx;
  G.y = d_y;
  G.y_mode = QMOE_Y_ACCUM_F32;
  G.ldy = ldy;
  G.bad = d_bad;
  general_matvec_kernel<<<std::max(1, (int)std::min<int64_t>((rows + 7) / 8, 4 * d->num_sms)), 256, 0, S(stream)>>>(G);
  CK(cudaGetLastError(), "general_matvec_kernel");
  return QMOE_OK;
}

int qmoe_fused_matvec(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, const uint32_t* d_mm,
                      int64_t rows, int64_t cols, const void* d_x, int x_dtype, float* d_y, int32_t* d_bad,
                      void* stream) {
  const int64_t ld = x_dtype == QMOE_X_BF16 ? ((cols + 7) / 8) * 8 : ((cols + 3) / 4) * 4;
  return fused_common(d, d_cw, d_row_off, d_mm, rows, cols, d_x, x_dtype, 1, ld, d_y, rows, d_bad, stream);
}

int qmoe_fused_matmat(qmoe_dict_t d, const uint16_t* d_cw, const int32_t* d_row_off, const uint32_t* d_mm,
                      int64_t rows, int64_t cols, const void* d_x, int x_dtype, int64_t ntok, int64_t ldx,
                      float* d_y, int64_t ldy, int32_t* d_bad, void* stream) {
  if (ldx < cols || ldy < rows) return qmoe::fail(QMOE_EINVAL, "leading dimension too small");
  return fused_common(d, d_cw, d_row_off, d_mm, rows, cols, d_x, x_dtype, ntok, ldx, d_y, ldy, d_bad, stream);
}

int qmoe_grouped_matvec(qmoe_dict_t d, const uint32_t* d_table, const qmoe_work* d_work, const int32_t* d_n_work,
                        int32_t max_work, int32_t max_cols, int32_t max_ntok, const void* d_x, int x_dtype,
                        int64_t ldx, void* d_y, int y_mode, int64_t ldy, int32_t* d_bad, void* stream) {
  if (!d || !d->d_stab || !d_work || !d_n_work || max_work < 0 || max_cols <= 0 || max_ntok < 1 ||
      max_ntok > QMOE_NT_MAX || (x_dtype != QMOE_X_F32 && x_dtype != QMOE_X_BF16) ||
      (y_mode != QMOE_Y_ACCUM_F32 && y_mode != QMOE_Y_RELU_BF16 && y_mode != QMOE_Y_STORE_F32))
    return qmoe::fail(QMOE_EINVAL, "bad argument");
  const int esz = x_dtype == QMOE_X_BF16 ? 2 : 4;
  if (!aligned16(d_x) || (ldx * esz) % 16) return qmoe::fail(QMOE_EINVAL, "x rows must be 16-byte aligned");
  if (max_work == 0) return QMOE_OK;
  if (d->sparse_ok) {
    if (max_ntok > NT_STREAM) return qmoe::fail(QMOE_EUNSUPPORTED, "streaming path takes <= 2 tokens per unit");
    StreamParams P{};
    P.gtab = pick_table(d, d_table, esz);
    P.work = d_work;
    P.n_work = d_n_work;
    P.max_work = max_work;
    P.x = d_x;
    P.ldx = ldx;
    P.y = d_y;
    P.y_mode = y_mode;
    P.ldy = ldy;
    P.bad = d_bad;
    return launch_stream(d, P, esz, max_cols, max_ntok, d->num_sms, QMOE_DICT_SIZE, S(stream));
  }
  if (d_table) return qmoe::fail(QMOE_EUNSUPPORTED, "codebooks need a <=3-non-zero dictionary");
  GeneralParams G{};
  G.words = d->d_words;
  G.work = d_work;
  G.n_work = d_n_work;
  G.max_work = max_work;
  G.x = d_x;
  G.x_bf16 = x_dtype == QMOE_X_BF16;
  G.ldx = ldx;
  G.y = d_y;
  G.y_mode = y_mode;
  G.ldy = ldy;
  G.bad = d_bad;
  general_matvec_kernel<<<4 * d->num_sms, 256, 0, S(stream)>>>(G);
  CK(cudaGetLastError(), "general_matvec_kernel");
  return QMOE_OK;
}

}  // extern "C"
