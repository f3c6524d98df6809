// Micro-benchmark of the decode+gather inner loop without the pipeline
// machinery (experiment, not product): lane per row, packed table prefix and
// x in shared memory, codewords read from global in 32-byte groups.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libubench.so tools/ubench.cu
#include <cstdint>
#include <cuda_runtime.h>

#define FULL 0xffffffffu

template <int MODE>
__global__ void __launch_bounds__(512, 1) ubench(const uint32_t* __restrict__ gtab, int H,
                                                 const uint16_t* __restrict__ cw, const int32_t* __restrict__ ro,
                                                 const uint32_t* __restrict__ mm, int rows, int cols,
                                                 const uint16_t* __restrict__ x, float* y) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* tab = sm;
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm + H);
  for (int i = threadIdx.x; i < H; i += blockDim.x) tab[i] = gtab[i];
  for (int i = threadIdx.x; i < cols + 64; i += blockDim.x) xs[i] = i < cols ? x[i] : 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int r0 = gw * 32; r0 < rows; r0 += nw * 32) {
    const int r = r0 + lane;
    int A = 0, B = 0;
    uint32_t m = 0;
    if (r < rows) { A = ro[r]; B = ro[r + 1]; m = mm[r]; }
    const float lmin = __uint_as_float(m << 16), lmax = __uint_as_float(m & 0xFFFF0000u);
    float acc = 0.f;
    int off = 0;
    const int g0 = A >> 4;
    const int ng = B > A ? ((B + 15) >> 4) - g0 : 0;
    const int maxg = __reduce_max_sync(FULL, ng);
    for (int g = 0; g < maxg; ++g) {
      const uint4* p = reinterpret_cast<const uint4*>(cw + (int64_t)(g0 + g) * 16);
      uint4 a = __ldg(p), b = __ldg(p + 1);
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      const int base = (g0 + g) * 16;
      const int lo = max(0, min(16, A - base)), hi = max(0, min(16, B - base));
      const uint32_t mask = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
      uint32_t t[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t c = (u & 1) ? (w[u >> 1] >> 16) : (w[u >> 1] & 0xFFFFu);
        const uint32_t e = c < (uint32_t)H ? tab[c] : __ldg(gtab + c);
        t[u] = ((mask >> u) & 1u) ? e : 0u;
      }
      if (MODE == 1) {  // lookups only (count lengths)
#pragma unroll
        for (int u = 0; u < 16; ++u) off += int(t[u] & 31u);
        continue;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const uint32_t e = t[u];
        const char* xo = reinterpret_cast<const char*>(xs + off);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const bool used = (e >> (26 + j)) & 1u;
          const float wv = ((e >> (29 + j)) & 1u) ? lmax : lmin;
          const uint16_t* xp = reinterpret_cast<const uint16_t*>(xo + ((e >> (5 + 7 * j)) & 0x7Fu));
          const float v = used ? __uint_as_float(uint32_t(*xp) << 16) : 0.f;
          acc = fmaf(wv, v, acc);
        }
        off += int(e & 31u);
      }
    }
    if (r < rows) y[r] = MODE == 1 ? (float)off : acc;
  }
}


// pipelined: group g+2 loaded, g+1 looked up, g applied
__device__ __forceinline__ void ldg2(const uint16_t* cw, int64_t g, uint4& a, uint4& b) {
  const uint4* p = reinterpret_cast<const uint4*>(cw + g * 16);
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(p));
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p + 1));
}
__device__ __forceinline__ void look(uint32_t (&t)[16], const uint4& a, const uint4& b, uint32_t mask, const uint32_t* tab,
                                     uint32_t H, const uint32_t* __restrict__ gtab) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const uint32_t c = (u & 1) ? (w[u >> 1] >> 16) : (w[u >> 1] & 0xFFFFu);
    const uint32_t e = c < H ? tab[c] : __ldg(gtab + c);
    t[u] = ((mask >> u) & 1u) ? e : 0u;
  }
}
__device__ __forceinline__ void app(const uint32_t (&t)[16], const uint16_t* xs, int& off, float lmin, float lmax, float& acc) {
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const uint32_t e = t[u];
    const char* xo = reinterpret_cast<const char*>(xs + off);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const bool used = (e >> (26 + j)) & 1u;
      const float wv = ((e >> (29 + j)) & 1u) ? lmax : lmin;
      const uint16_t* xp = reinterpret_cast<const uint16_t*>(xo + ((e >> (5 + 7 * j)) & 0x7Fu));
      const float v = used ? __uint_as_float(uint32_t(*xp) << 16) : 0.f;
      acc = fmaf(wv, v, acc);
    }
    off += int(e & 31u);
  }
}
__device__ __forceinline__ uint32_t gmask(int64_t g, int A, int B) {
  const int64_t base = g * 16;
  const int lo = (int)max((int64_t)0, min((int64_t)16, A - base));
  const int hi = (int)max((int64_t)0, min((int64_t)16, B - base));
  return ((1u << hi) - 1u) & ~((1u << lo) - 1u);
}
__global__ void __launch_bounds__(512, 1) ubench_pipe(const uint32_t* __restrict__ gtab, int H,
                                                      const uint16_t* __restrict__ cw, const int32_t* __restrict__ ro,
                                                      const uint32_t* __restrict__ mm, int rows, int cols,
                                                      const uint16_t* __restrict__ x, float* y) {
  extern __shared__ __align__(16) uint32_t sm[];
  uint32_t* tab = sm;
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm + H);
  for (int i = threadIdx.x; i < H; i += blockDim.x) tab[i] = gtab[i];
  for (int i = threadIdx.x; i < cols + 64; i += blockDim.x) xs[i] = i < cols ? x[i] : 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int r0 = gw * 32; r0 < rows; r0 += nw * 32) {
    const int r = r0 + lane;
    int A = 0, B = 0;
    uint32_t m = 0;
    if (r < rows) { A = ro[r]; B = ro[r + 1]; m = mm[r]; }
    const float lmin = __uint_as_float(m << 16), lmax = __uint_as_float(m & 0xFFFF0000u);
    float acc = 0.f;
    int off = 0;
    const int64_t g0 = A >> 4;
    const int ng = B > A ? ((B + 15) >> 4) - (int)g0 : 0;
    const int maxg = __reduce_max_sync(FULL, ng);
    if (maxg > 0) {
      uint4 ra0, ra1, rb0, rb1;
      uint32_t ta[16], tb[16];
      ldg2(cw, g0, ra0, ra1);
      if (maxg > 1) ldg2(cw, g0 + 1, rb0, rb1);
      look(ta, ra0, ra1, gmask(g0, A, B), tab, H, gtab);
      for (int it = 0;;) {
        if (it + 2 < maxg) ldg2(cw, g0 + it + 2, ra0, ra1);
        if (it + 1 < maxg) look(tb, rb0, rb1, gmask(g0 + it + 1, A, B), tab, H, gtab);
        app(ta, xs, off, lmin, lmax, acc);
        if (++it >= maxg) break;
        if (it + 2 < maxg) ldg2(cw, g0 + it + 2, rb0, rb1);
        if (it + 1 < maxg) look(ta, ra0, ra1, gmask(g0 + it + 1, A, B), tab, H, gtab);
        app(tb, xs, off, lmin, lmax, acc);
        if (++it >= maxg) break;
      }
    }
    if (r < rows) y[r] = acc;
  }
}

extern "C" int ubench_run(int mode, const uint32_t* gtab, int H, const uint16_t* cw, const int32_t* ro,
                          const uint32_t* mm, int rows, int cols, const uint16_t* x, float* y, int grid,
                          void* stream) {
  const size_t smem = (size_t)H * 4 + (cols + 64) * 2;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (mode == 2) {
    cudaFuncSetAttribute(ubench_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ubench_pipe<<<grid, 512, smem, s>>>(gtab, H, cw, ro, mm, rows, cols, x, y);
  } else if (mode == 1) {
    cudaFuncSetAttribute(ubench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ubench<1><<<grid, 512, smem, s>>>(gtab, H, cw, ro, mm, rows, cols, x, y);
  } else {
    cudaFuncSetAttribute(ubench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ubench<0><<<grid, 512, smem, s>>>(gtab, H, cw, ro, mm, rows, cols, x, y);
  }
  return (int)cudaGetLastError();
}
