// Internal declarations shared by the host (.cpp) and device (.cu) halves.
#pragma once
#include <cstdint>
#include <string>

namespace qmoe {

int fail(int code, const std::string& msg);
const char* last_error();

int generate_words(double p0, uint32_t* words);
int unpack_entry(const uint32_t* words, int i, int* n_out, uint8_t* vals);
int build_trie(const uint32_t* words, int32_t* next_node, int32_t* entry_of_node);

// Kernel-private tables derived from the decode words (built once per dictionary):
//  sparse_tab[e]: bits 0-4 = 2n (values in the entry), bits 5-6 = min(nnz, 3),
//                 byte k+1 (k = 0..2) = k-th non-zero value: bit0 code 1, bit1 code 2,
//                 bits 2-6 its position in the entry (0..27). Valid when max_nz <= 3.
//  len_tab[e]:    2n
int derive_tables(const uint32_t* words, uint32_t* sparse_tab, uint8_t* len_tab, int* max_nz);

// Matvec-format tables, two variants back to back, MT_STRIDE entries each
// (entries from 65536 are padding). Valid when max_nz <= 3.
//   variant 0 (packed fields; decompress, checkpoints): bits 0-4 len = 2n |
//     bits 5-11/12-18/19-25 4*position of non-zero 0..2 | bits 26-28 used |
//     bits 29-31 code 2.
//   variant 1 (byte fields; streaming matvec): byte j = 4*position of
//     non-zero j or 0x7F (unused) | bits 24-26 code 2 | bits 28-31 n.
// Stride 65540 keeps the second variant 16-byte aligned.
constexpr int MT_STRIDE = 65540;
int derive_matvec_tables(const uint32_t* sparse_tab, uint32_t* mtab /* 2 * MT_STRIDE */);

}  // namespace qmoe
