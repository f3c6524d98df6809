// Host half of libqmoe: dictionary generation, trie rebuild and the derivation
// of the kernel-private tables. No CUDA calls here, so these entry points work
// on a CPU-only machine (the CPU test-suite exercises them).
//
// Reference semantics (paths relative to /root/reference/pkg/src/moepack/):
//   generate_dictionary  dictionary.py:234-279  best-first heap, key (-logp, n, bytes)
//   _pack_all            dictionary.py:137-147  word w = n | v[14w+i] << (4+2i)
//   _unpack_all          dictionary.py:150-167  validation rules
//   _build_trie          dictionary.py:170-194  parents-first, prefix-closed
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <string>
#include <vector>

#include "qmoe.h"
#include "qmoe_internal.h"

namespace qmoe {

static thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

const char* last_error() { return g_err.c_str(); }

namespace {

// One candidate sequence on the best-first frontier. `vals` holds the 2n
// ternary values; ordering below reproduces Python's tuple ordering of the
// reference heap items (-logp, n_pairs, value bytes, parent, zeros).
struct Cand {
  double neg_logp;
  int n;
  int parent;
  int zeros;
  uint8_t vals[28];
};

struct CandGreater {
  bool operator()(const Cand& a, const Cand& b) const {
    if (a.neg_logp != b.neg_logp) return a.neg_logp > b.neg_logp;
    if (a.n != b.n) return a.n > b.n;
    int c = std::memcmp(a.vals, b.vals, 2 * a.n);  // equal n => equal length
    if (c != 0) return c > 0;
    if (a.parent != b.parent) return a.parent > b.parent;
    return a.zeros > b.zeros;
  }
};

}  // namespace

int generate_words(double p0, uint32_t* words) {
  if (!(p0 > 1.0 / 3.0 && p0 < 1.0))
    return fail(QMOE_EINVAL, "dictionary generation requires 1/3 < p0 < 1");
  // Written so the compiler cannot contract into FMA: the heap keys must be
  // bit-identical to the reference's float64 arithmetic.
  volatile double lp0 = std::log(p0);
  volatile double lq = std::log((1.0 - p0) / 2.0);
  std::priority_queue<Cand, std::vector<Cand>, CandGreater> heap;
  Cand root{};
  root.neg_logp = -0.0;
  root.n = 0;
  root.parent = -1;
  root.zeros = 0;
  heap.push(root);
  std::vector<uint8_t> vals(size_t(QMOE_DICT_SIZE) * 28, 0);
  std::vector<uint8_t> npairs(QMOE_DICT_SIZE, 0);
  int filled = 0;
  while (filled < QMOE_DICT_SIZE) {
    Cand c = heap.top();
    heap.pop();
    int me = -1;
    if (c.n > 0) {
      me = filled++;
      npairs[me] = uint8_t(c.n);
      std::memcpy(&vals[size_t(me) * 28], c.vals, 2 * c.n);
    }
    if (c.n >= QMOE_MAX_PAIRS) continue;
    for (int a = 0; a < 3; ++a) {
      for (int b = 0; b < 3; ++b) {
        Cand ch;
        ch.n = c.n + 1;
        ch.parent = me;
        ch.zeros = c.zeros + (a == 0) + (b == 0);
        int nonzeros = 2 * ch.n - ch.zeros;
        volatile double t0 = double(ch.zeros) * lp0;
        volatile double t1 = double(nonzeros) * lq;
        volatile double logp = t0 + t1;
        ch.neg_logp = -logp;
        std::memset(ch.vals, 0, sizeof ch.vals);
        std::memcpy(ch.vals, c.vals, 2 * c.n);
        ch.vals[2 * c.n] = uint8_t(a);
        ch.vals[2 * c.n + 1] = uint8_t(b);
        heap.push(ch);
      }
    }
  }
  for (int i = 0; i < QMOE_DICT_SIZE; ++i) {
    uint32_t w[2] = {npairs[i], npairs[i]};
    for (int v = 0; v < 2 * npairs[i]; ++v)
      w[v / 14] |= uint32_t(vals[size_t(i) * 28 + v]) << (4 + 2 * (v % 14));
    words[2 * i] = w[0];
    words[2 * i + 1] = w[1];
  }
  return QMOE_OK;
}

int unpack_entry(const uint32_t* words, int i, int* n_out, uint8_t* vals) {
  uint32_t w0 = words[2 * i], w1 = words[2 * i + 1];
  int n = int(w0 & 0xF);
  if (n != int(w1 & 0xF)) return fail(QMOE_ECORRUPT, "pair counts differ between decode words");
  if (n < 1 || n > QMOE_MAX_PAIRS) return fail(QMOE_ECORRUPT, "pair count out of range in decode words");
  for (int v = 0; v < 28; ++v) {
    uint32_t w = v < 14 ? w0 : w1;
    uint8_t code = uint8_t((w >> (4 + 2 * (v % 14))) & 3u);
    if (v >= 2 * n && code != 0) return fail(QMOE_ECORRUPT, "non-zero padding in decode words");
    vals[v] = code;
  }
  *n_out = n;
  return QMOE_OK;
}

int build_trie(const uint32_t* words, int32_t* next_node, int32_t* entry_of_node) {
  const int n = QMOE_DICT_SIZE;
  for (size_t i = 0; i < size_t(n + 1) * 9; ++i) next_node[i] = -1;
  for (int i = 0; i <= n; ++i) entry_of_node[i] = -1;
  uint8_t vals[28];
  for (int i = 0; i < n; ++i) {
    int np = 0;
    int rc = unpack_entry(words, i, &np, vals);
    if (rc) return rc;
    int node = 0;
    for (int j = 0; j + 1 < np; ++j) {
      node = next_node[size_t(node) * 9 + 3 * vals[2 * j] + vals[2 * j + 1]];
      if (node < 0) return fail(QMOE_ECORRUPT, "entry table is not prefix-closed");
    }
    int sym = 3 * vals[2 * np - 2] + vals[2 * np - 1];
    int32_t& slot = next_node[size_t(node) * 9 + sym];
    if (slot != -1) return fail(QMOE_ECORRUPT, "duplicate entry in table");
    slot = i + 1;
    entry_of_node[i + 1] = i;
  }
  for (int s = 0; s < 9; ++s)
    if (next_node[s] < 0) return fail(QMOE_ECORRUPT, "dictionary must contain all nine single pairs");
  return QMOE_OK;
}

int derive_tables(const uint32_t* words, uint32_t* sparse_tab, uint8_t* len_tab, int* max_nz) {
  uint8_t vals[28];
  int mx = 0;
  for (int i = 0; i < QMOE_DICT_SIZE; ++i) {
    int np = 0;
    int rc = unpack_entry(words, i, &np, vals);
    if (rc) return rc;
    len_tab[i] = uint8_t(2 * np);
    uint32_t e = uint32_t(2 * np);  // bits 0-4: values in the entry
    int nz = 0;
    for (int v = 0; v < 2 * np; ++v) {
      if (!vals[v]) continue;
      if (nz < 3) {
        // slot byte: bit0 = code 1 (row min), bit1 = code 2 (row max), bits 2-6 = position
        uint32_t slot = (vals[v] == 1 ? 1u : 2u) | (uint32_t(v) << 2);
        e |= slot << (8 * (nz + 1));
      }
      ++nz;
    }
    e |= uint32_t(nz < 3 ? nz : 3) << 5;
    if (nz > mx) mx = nz;
    sparse_tab[i] = e;
  }
  *max_nz = mx;
  return QMOE_OK;
}

int derive_matvec_tables(const uint32_t* sparse_tab, uint32_t* mtab) {
  // variant 0: packed-field format (decompress / checkpoints)
  uint32_t* t = mtab;
  for (int i = 0; i < QMOE_DICT_SIZE; ++i) {
    const uint32_t e = sparse_tab[i];
    uint32_t m = e & 31u;
    for (int j = 0; j < 3; ++j) {
      const uint32_t b = (e >> (8 * (j + 1))) & 0xFFu;
      if (!b) continue;
      m |= ((b >> 2) * 4u) << (5 + 7 * j);
      m |= 1u << (26 + j);
      if (b & 2u) m |= 1u << (29 + j);
    }
    t[i] = m;
  }
  for (int i = QMOE_DICT_SIZE; i < MT_STRIDE; ++i) t[i] = 0;
  // variant 1: byte-field "segment" format of the streaming matvec: byte j
  // (j = 0..2) = 4 * position of non-zero j (0x7F: slot unused), bits 24-26
  // = non-zero j is code 2 (row max), bits 28-31 = n (pairs; 2n values).
  t = mtab + MT_STRIDE;
  for (int i = 0; i < QMOE_DICT_SIZE; ++i) {
    const uint32_t e = sparse_tab[i];
    uint32_t m = ((e & 31u) >> 1) << 28;
    for (int j = 0; j < 3; ++j) {
      const uint32_t b = (e >> (8 * (j + 1))) & 0xFFu;
      if (!b) {
        m |= 0x7Fu << (8 * j);
        continue;
      }
      m |= ((b >> 2) * 4u) << (8 * j);
      if (b & 2u) m |= 1u << (24 + j);
    }
    t[i] = m;
  }
  for (int i = QMOE_DICT_SIZE; i < MT_STRIDE; ++i) t[i] = 0x007F7F7Fu;
  return QMOE_OK;
}

}  // namespace qmoe

extern "C" {

const char* qmoe_version(void) { return "qmoe-b200 0.1 (sm_100a)"; }
const char* qmoe_last_error(void) { return qmoe::last_error(); }

int qmoe_generate_decode_words(double p0, uint32_t* h_words) {
  if (!h_words) return qmoe::fail(QMOE_EINVAL, "null output");
  return qmoe::generate_words(p0, h_words);
}

int qmoe_build_trie(const uint32_t* h_words, int32_t* h_next_node, int32_t* h_entry_of_node) {
  if (!h_words || !h_next_node || !h_entry_of_node) return qmoe::fail(QMOE_EINVAL, "null argument");
  return qmoe::build_trie(h_words, h_next_node, h_entry_of_node);
}

}  // extern "C"
