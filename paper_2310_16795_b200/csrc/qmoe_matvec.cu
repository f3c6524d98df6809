// Fused dictionary-decode + matvec (codec.py:196-244 semantics) for sm_100a.
//
// lean_matvec_kernel — the product path for dictionaries whose entries hold
// <= 3 non-zero values (the default p0 = 0.885 dictionary):
//   * persistent, one CTA per SM; the CTA takes a contiguous slice of the work
//     list and merges consecutive units that share their x rows (they are row
//     blocks of one matrix for one token chunk — qmoe_moe_plan's order) into
//     one RUN: x is staged once per run, then the 16 warps stride over the
//     run's row tasks with no further CTA synchronisation;
//   * the hot prefix of the packed entry table (a frequency codebook in the
//     MoE layer) is staged in shared memory once per launch;
//   * a task is 32 / G rows: each lane owns one contiguous SEGMENT of a row
//     (G = 2^lg segments, lg from the matrix's checkpoints; lg = 0: a lane per
//     row) and walks it with a running column offset starting at the row's
//     checkpoint — no scans. Codewords stream from HBM in sector-aligned
//     16-codeword groups (2 x 16-byte loads bypassing L1), group g+2 loaded,
//     g+1 looked up and g applied per iteration; the next task's row
//     metadata is prefetched while the current task runs;
//   * per non-zero slot acc += level(code) * x[col] in fp32; the row's sum is
//     reduced over its G lanes and bf16-rounded once (codec.py:243).
// Entry format "matvec" (qmoe_host.cpp, esz = bytes per staged x element):
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

#ifndef QMOE_LEAN_THREADS
#define QMOE_LEAN_THREADS 512
#endif
constexpr int THREADS = QMOE_LEAN_THREADS;
constexpr int NWARPS = THREADS / 32;
constexpr int GRP = 16;                // codewords per aligned 32-byte group
constexpr int NT_STREAM = 2;           // tokens per unit on the streaming path
constexpr int MAX_LG = 2;              // G <= 4 lanes per row on the fast path

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

struct Rec {  // == qmoe_work (80 bytes)
  const uint16_t* cw;
  const int32_t* ro;
  const uint32_t* mm;
  const uint16_t* ck;
  int32_t cols, row0, row1, ntok, cw0, cw1, lg, pad;
  int32_t tok[QMOE_NT_MAX];
};
static_assert(sizeof(Rec) == sizeof(qmoe_work), "record layout");

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
  int xcap;                   // elements per token slot of the x buffer
  int ntmax;                  // token slots
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
    R.cw0 = 0;
    R.cw1 = 0;
  }
}

// same matrix, contiguous rows and same tokens: the units merge into one run
__device__ __forceinline__ bool continues(const Rec& a, const Rec& b) {
  bool s = a.cw == b.cw && a.row1 == b.row0 && a.ntok == b.ntok && a.lg == b.lg;
#pragma unroll
  for (int q = 0; q < QMOE_NT_MAX; ++q) s = s && (q >= a.ntok || a.tok[q] == b.tok[q]);
  return s;
}

__device__ __forceinline__ void ld_group(const uint16_t* cw, int64_t g, uint4& a, uint4& b) {
  const uint4* p = reinterpret_cast<const uint4*>(cw + g * GRP);
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w)
               : "l"(p));
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p + 1));
}

// entries of the 16 codewords of a group; positions outside the lane's
// segment (mask bit clear) get the zero entry
__device__ __forceinline__ void lookup_group(uint32_t (&t)[GRP], const uint4& a, const uint4& b, uint32_t mask,
                                             const uint32_t* tab, uint32_t H, const uint32_t* __restrict__ gtab) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int u = 0; u < GRP; ++u) {
    const uint32_t c = (u & 1) ? (w[u >> 1] >> 16) : (w[u >> 1] & 0xFFFFu);
    const uint32_t e = c < H ? tab[c] : __ldg(gtab + c);
    t[u] = ((mask >> u) & 1u) ? e : 0u;
  }
}

template <int NT, int ESZ>
__device__ __forceinline__ void apply_group(const uint32_t (&t)[GRP], const typename XType<ESZ>::T* xs, int xslot,
                                            int& off, float lmin, float lmax, float (&acc)[NT]) {
  using XT = typename XType<ESZ>::T;
#pragma unroll
  for (int u = 0; u < GRP; ++u) {
    const uint32_t e = t[u];
    const char* xo = reinterpret_cast<const char*>(xs + off);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const bool used = (e >> (26 + j)) & 1u;
      const float w = ((e >> (29 + j)) & 1u) ? lmax : lmin;
      const XT* xp = reinterpret_cast<const XT*>(xo + ((e >> (5 + 7 * j)) & 0x7Fu));
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const float v = used ? XType<ESZ>::get(xp[q * xslot]) : 0.f;
        acc[q] = fmaf(w, v, acc[q]);
      }
    }
    off += int(e & 31u);
  }
}

__device__ __forceinline__ uint32_t group_mask(int64_t g, int64_t A, int64_t B) {
  const int64_t base = g * GRP;
  const int lo = (int)max((int64_t)0, min((int64_t)GRP, A - base));
  const int hi = (int)max((int64_t)0, min((int64_t)GRP, B - base));
  return ((1u << hi) - 1u) & ~((1u << lo) - 1u);
}

// row metadata of one lane's segment
struct Seg {
  int64_t A, B;  // codeword range
  int off;       // starting column
  uint32_t mm;   // bf16 (min, max)
  int row;       // absolute row, or -1
};

__device__ __forceinline__ Seg load_seg(const Rec& R, int task, int lg, int rb) {
  Seg sg{0, 0, 0, 0u, -1};
  const int lane = threadIdx.x & 31;
  const int G = 1 << lg;
  const int r = R.row0 + (task << (5 - lg)) + (lane >> lg);
  if (r < rb) {
    const int seg = lane & (G - 1);
    const int s = __ldg(R.ro + r), e = __ldg(R.ro + r + 1);
    const int n = e - s;
    sg.A = s + ((seg * n) >> lg);
    sg.B = s + (((seg + 1) * n) >> lg);
    sg.off = seg ? (int)__ldg(R.ck + (size_t)r * (G - 1) + seg - 1) : 0;
    sg.mm = __ldg(R.mm + r);
    sg.row = r;
  }
  return sg;
}

template <int NT, int ESZ>
__device__ __forceinline__ void run_task(const StreamParams& P, const Rec& R, const Seg& sg, int lg, const int (&tok)[NT],
                                         const typename XType<ESZ>::T* xs, const uint32_t* tab) {
  const int lane = threadIdx.x & 31;
  const int G = 1 << lg;
  const uint32_t H = (uint32_t)P.H;
  const uint32_t* gtab = P.gtab;
  const int64_t A = sg.A, B = sg.B;
  const bool has = sg.row >= 0 && B > A;
  const int64_t g0 = has ? A / GRP : 0;
  const int ng = has ? (int)((B + GRP - 1) / GRP - g0) : 0;
  const int64_t glast = has ? (B - 1) / GRP : 0;
  const int maxg = __reduce_max_sync(FULL_MASK, ng);
  const float lmin = __uint_as_float(sg.mm << 16), lmax = __uint_as_float(sg.mm & 0xFFFF0000u);
  int off = sg.off;
  float acc[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) acc[q] = 0.f;
  if (maxg > 0) {
    const uint16_t* cw = R.cw;
    uint4 ra0, ra1, rb0, rb1;
    uint32_t ta[GRP], tb[GRP];
    // groups past this lane's segment re-read its last group (mask 0)
    ld_group(cw, g0, ra0, ra1);
    if (maxg > 1) ld_group(cw, min(g0 + 1, glast), rb0, rb1);
    lookup_group(ta, ra0, ra1, group_mask(g0, A, B), tab, H, gtab);
    for (int it = 0;;) {
      if (it + 2 < maxg) ld_group(cw, min(g0 + it + 2, glast), ra0, ra1);
      if (it + 1 < maxg) lookup_group(tb, rb0, rb1, group_mask(g0 + it + 1, A, B), tab, H, gtab);
      apply_group<NT, ESZ>(ta, xs, P.xcap, off, lmin, lmax, acc);
      if (++it >= maxg) break;
      if (it + 2 < maxg) ld_group(cw, min(g0 + it + 2, glast), rb0, rb1);
      if (it + 1 < maxg) lookup_group(ta, ra0, ra1, group_mask(g0 + it + 1, A, B), tab, H, gtab);
      apply_group<NT, ESZ>(tb, xs, P.xcap, off, lmin, lmax, acc);
      if (++it >= maxg) break;
    }
  }
#pragma unroll
  for (int q = 0; q < NT; ++q) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
      if (d < G) acc[q] += __shfl_xor_sync(FULL_MASK, acc[q], d);
  }
  if (sg.row < 0 || (lane & (G - 1)) != G - 1) return;  // the last segment's lane ends the row
  const int r = sg.row;
  if (off != R.cols) {  // row decodes to the wrong number of values: never written
    if (P.bad) {
      atomicAdd(P.bad, 1);
      atomicMin(P.bad + 1, r);
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    if (q >= R.ntok) break;
    const float v = bf16_round_dev(acc[q]);
    if (P.y_mode == QMOE_Y_RELU_BF16) {
      reinterpret_cast<uint16_t*>(P.y)[(int64_t)tok[q] * P.ldy + r] = (uint16_t)(__float_as_uint(fmaxf(v, 0.f)) >> 16);
    } else if (P.y_mode == QMOE_Y_STORE_F32) {
      reinterpret_cast<float*>(P.y)[(int64_t)tok[q] * P.ldy + r] = v + 0.f;  // == 0 + v
    } else {
      float* yp = reinterpret_cast<float*>(P.y) + (int64_t)tok[q] * P.ldy + r;
      *yp = *yp + v;
    }
  }
}

// the warp's tasks of one run: task = warp, warp + NWARPS, ... with the next
// task's segment metadata loaded before the current task runs
template <int NT, int ESZ>
__device__ __forceinline__ void run_run(const StreamParams& P, const Rec& R, int rb, const typename XType<ESZ>::T* xs,
                                        const uint32_t* tab) {
  const int warp = threadIdx.x >> 5;
  const int lg = R.lg;
  const int ntasks = (rb - R.row0 + (32 >> lg) - 1) >> (5 - lg);
  int tok[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) tok[q] = R.tok[q];
  int task = warp;
  if (task >= ntasks) return;
  Seg cur = load_seg(R, task, lg, rb);
  for (;;) {
    const int nt = task + NWARPS;
    Seg nxt{0, 0, 0, 0u, -1};
    if (nt < ntasks) nxt = load_seg(R, nt, lg, rb);
    run_task<NT, ESZ>(P, R, cur, lg, tok, xs, tab);
    if (nt >= ntasks) break;
    cur = nxt;
    task = nt;
  }
}

// x is always staged as fp32 (converted while copying), so the inner loop
// uses the esz-4 entry table and needs no per-slot conversion.
template <int IN_ESZ>
__global__ void __launch_bounds__(THREADS, 1) lean_matvec_kernel(StreamParams P) {
  constexpr int ESZ = 4;
  using XT = float;
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem);
  XT* xs = reinterpret_cast<XT*>(smem + (size_t)P.H * 4);
  __shared__ int s_run_end;
  __shared__ Rec s_rec;

  int n;
  if (P.work) n = min(*P.n_work, P.max_work);
  else {
    const int nblk = (P.single.rows + P.rows_per_unit - 1) / P.rows_per_unit;
    n = nblk * (int)((P.ntok_single + P.ntu_single - 1) / P.ntu_single);
  }
  const int u0 = (int)((int64_t)n * blockIdx.x / gridDim.x);
  const int u1 = (int)((int64_t)n * (blockIdx.x + 1) / gridDim.x);
  if (u0 >= u1) return;
  {  // table prefix: vectorised copy by all threads
    const uint4* src = reinterpret_cast<const uint4*>(P.gtab);
    uint4* dst = reinterpret_cast<uint4*>(tab);
    for (int i = threadIdx.x; i < P.H / 4; i += THREADS) dst[i] = __ldg(src + i);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int u = u0; u < u1;) {
    // ---- find the run starting at u (warp 0: 32 records per step)
    if (warp == 0) {
      Rec first;
      make_rec(P, u, first);
      int end = u + 1;
      bool open = true;
      for (int base = u + 1; open && base < u1; base += 31) {
        // lane j (j >= 1) checks unit base + j - 1 against its predecessor
        Rec mine, prev;
        const int v = base + lane - 1;
        if (lane >= 1 && v < u1) {
          make_rec(P, v, mine);
          make_rec(P, v - 1, prev);
        }
        const bool ok = lane >= 1 && v < u1 && continues(prev, mine);
        const unsigned brk = __ballot_sync(FULL_MASK, !ok) & ~1u;
        if (brk) {
          end = base + (__ffs(brk) - 1) - 1;
          open = false;
        } else {
          end = min(u1, base + 31);
        }
      }
      if (lane == 0) {
        s_run_end = end;
        s_rec = first;
      }
    }
    __syncthreads();  // previous run finished (x buffer free) + run published
    const int end = s_run_end;
    Rec R = s_rec;
    if (end - 1 > u) {
      Rec last;
      make_rec(P, end - 1, last);
      R.cw1 = last.cw1;
      R.row1 = last.row1;
    }
    if (!P.work) R.cw1 = 0;
    // ---- stage x rows of the run's tokens
    for (int q = 0; q < R.ntok; ++q) {
      XT* dst = xs + (size_t)q * P.xcap;
      if (IN_ESZ == 2) {
        const uint16_t* src = reinterpret_cast<const uint16_t*>(P.x) + (int64_t)R.tok[q] * P.ldx;
        for (int i = threadIdx.x; i < P.xcap; i += THREADS)
          dst[i] = i < R.cols ? __uint_as_float(uint32_t(__ldg(src + i)) << 16) : 0.f;
      } else {
        const float* src = reinterpret_cast<const float*>(P.x) + (int64_t)R.tok[q] * P.ldx;
        for (int i = threadIdx.x; i < P.xcap; i += THREADS) dst[i] = i < R.cols ? __ldg(src + i) : 0.f;
      }
    }
    __syncthreads();
    if (R.ntok == 1) run_run<1, ESZ>(P, R, R.row1, xs, tab);
    else run_run<2, ESZ>(P, R, R.row1, xs, tab);
    u = end;
  }
}

// ----------------------------------------------------------------- host side
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int hot_override() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("QMOE_HOT_ENTRIES");
    v = e ? atoi(e) : -1;
  }
  return v;
}

int launch_lean(const qmoe_dict* d, StreamParams& P, int esz, int max_cols, int ntmax, int grid, int hot_want,
                cudaStream_t st) {
  P.ntmax = ntmax;
  P.xcap = ((max_cols + 32 + 15) / 16) * 16;
  const size_t xbytes = (size_t)ntmax * P.xcap * 4;  // staged as fp32
  const size_t static_smem = sizeof(Rec) + 64;
  if (xbytes + static_smem + 4096 > (size_t)d->max_smem_optin)
    return qmoe::fail(QMOE_EUNSUPPORTED, "cols too large for the shared-memory x staging buffer");
  int H = (int)((d->max_smem_optin - xbytes - static_smem - 256) / 4);
  if (hot_override() >= 0) hot_want = hot_override();
  H = std::min(H, std::min(hot_want, QMOE_DICT_SIZE));
  H &= ~255;
  P.H = H;
  const size_t smem = (size_t)H * 4 + xbytes;
  if (esz == 2) {
    CK(cudaFuncSetAttribute(lean_matvec_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    lean_matvec_kernel<2><<<grid, THREADS, smem, st>>>(P);
  } else {
    CK(cudaFuncSetAttribute(lean_matvec_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
    lean_matvec_kernel<4><<<grid, THREADS, smem, st>>>(P);
  }
  CK(cudaGetLastError(), "lean_matvec_kernel launch");
  return QMOE_OK;
}

const uint32_t* pick_table(const qmoe_dict* d, const uint32_t* user, int esz) {
  // tables hold both variants back to back: [esz 4 | esz 2], MT_STRIDE entries each
  if (user) return esz == 4 ? user : user + qmoe::MT_STRIDE;
  return esz == 4 ? d->d_mtab : d->d_mtab + qmoe::MT_STRIDE;
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
    const int rpu = 256;
    const int ntu = (int)std::min<int64_t>(ntok, NT_STREAM);
    StreamParams P{};
    P.gtab = pick_table(d, nullptr, 4);  // x is staged as fp32
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
    return launch_lean(d, P, esz, (int)cols, ntu, grid, want, S(stream));
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
    P.gtab = pick_table(d, d_table, 4);  // x is staged as fp32
    P.work = d_work;
    P.n_work = d_n_work;
    P.max_work = max_work;
    P.x = d_x;
    P.ldx = ldx;
    P.y = d_y;
    P.y_mode = y_mode;
    P.ldy = ldy;
    P.bad = d_bad;
    return launch_lean(d, P, esz, max_cols, max_ntok, d->num_sms, QMOE_DICT_SIZE, S(stream));
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
