/*
 * qmoe.h — C-ABI of the B200-native QMoE compressed decode + matvec library
 * (libqmoe.so, built from paper_2310_16795_b200/csrc/).
 *
 * The reference (`moepack`, pure Python/numpy) has no FFI: its boundary is the
 * Python operator API in /root/reference/pkg/src/moepack/codec.py. Every
 * entry point below replaces one reference function; the citation is given on
 * each declaration (paths relative to /root/reference/pkg/src/moepack/).
 * INTEGRATION.md shows the ctypes binding a moepack maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only. Pointers marked d_ are DEVICE pointers,
 *    h_ are HOST pointers. `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream). Device calls are asynchronous on `stream`
 *    and never allocate on the hot path (dictionary handles own their tables).
 *  - Return status: QMOE_OK, QMOE_EINVAL (bad argument / shape),
 *    QMOE_ECORRUPT (data failed validation; host-side checks only — device-side
 *    corruption is reported through d_bad), QMOE_ECUDA (CUDA launch/runtime
 *    error), QMOE_EUNSUPPORTED. qmoe_last_error() returns a thread-local
 *    message for the last non-OK status.
 *  - Compressed matrix layout (CompressedMatrix, codec.py:33-60):
 *      cw        uint16[n_cw]        codeword stream, row r owns [row_off[r], row_off[r+1])
 *      row_off   int32[rows + 1]     monotone, row_off[0] = 0, row_off[rows] = n_cw
 *      row_minmax uint32[rows]       bf16 pair: low half = min bits, high half = max bits
 *                                     (== uint16 (rows, 2) little-endian)
 *  - y semantics of every matvec (codec.py:242-243):
 *      y[r] += bf16_rne( fp32 sum_j level(code[r][j]) * x[j] ),  y float32,
 *      level(0) = 0, level(1) = f32(bf16 min), level(2) = f32(bf16 max).
 */
#ifndef QMOE_H_
#define QMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  QMOE_OK = 0,
  QMOE_EINVAL = 1,
  QMOE_ECORRUPT = 2,
  QMOE_ECUDA = 3,
  QMOE_EUNSUPPORTED = 4
};

enum { QMOE_X_F32 = 0, QMOE_X_BF16 = 1 };

#define QMOE_DICT_SIZE 65536
#define QMOE_MAX_PAIRS 14
#define QMOE_NT_MAX 4 /* tokens per grouped work unit (inner token loop) */

typedef struct qmoe_dict* qmoe_dict_t;

/* One compressed matrix resident on the device (grouped launches): the
 * reference format (cw / row_off / row_minmax as in CompressedMatrix; the
 * arrays must start 16-byte aligned and be readable 32 bytes past their end)
 * plus optional kernel-private, read-only derived data:
 *  ck / lg: row-segment checkpoints (qmoe_checkpoints): with G = 2^lg lanes
 *    per row, ck[r * (G-1) + j - 1] is the column at which segment j of row r
 *    starts; segment j starts at codeword s + j*n/G rounded UP to a multiple
 *    of 8 (clamped to the row end e), so inner segment boundaries are 16-byte
 *    group boundaries of the stream.
 *  row_id, colpts: reserved, must be NULL. */
typedef struct qmoe_matrix {
  const uint16_t* cw;
  const int32_t* row_off;
  const uint32_t* row_minmax;
  const uint16_t* ck;
  int32_t rows;
  int32_t cols;
  int32_t n_cw;
  int32_t lg;
  const uint16_t* row_id;
  const uint32_t* colpts;
} qmoe_matrix;

/* One RUN of a grouped launch (self-contained, 80 bytes): rows [row0, row1)
 * of one matrix (fields as qmoe_matrix; row_id reserved, NULL), applied to `ntok` tokens (<= 2
 * on the streaming path) with G = 2^lg lanes per row. Token t reads x row
 * tok[t] (x + tok[t] * ldx) and writes y row tok[t] (y + tok[t] * ldy). A
 * run is cut into ceil(((row1 - row0) << lg) / 32) warp TASKS; task0 is the
 * exclusive prefix of those counts over the list (the launch splits the
 * global task range evenly over the SMs). Written by qmoe_moe_plan (or by
 * the caller). */
typedef struct qmoe_work {
  const uint16_t* cw;
  const int32_t* row_off;
  const uint32_t* row_minmax;
  const uint16_t* ck;
  int32_t cols;
  int32_t row0;
  int32_t row1;
  int32_t lg;
  int32_t ntok;
  int32_t task0;
  const uint16_t* row_id;
  int32_t tok[QMOE_NT_MAX];
} qmoe_work;

/* y modes of the grouped launch */
enum {
  QMOE_Y_ACCUM_F32 = 0,     /* y (f32) += bf16(dot)                       (codec.py:243) */
  QMOE_Y_RELU_BF16 = 1,     /* y (bf16) = relu(bf16(dot)) — the FFN hidden h, written
                               once from zero: equals relu(fused_matvec(wi, x, y=0)) */
  QMOE_Y_STORE_F32 = 2,     /* y (f32) = 0 + bf16(dot): accumulate into a zero y
                               without reading it */
  QMOE_Y_RESID_BF16 = 3     /* fused step only (qmoe_moe_step_resid): y (bf16) =
                               bf16(x + gate * bf16(dot)), the layer's residual add */
};

/* ------------------------------------------------------------------ host-only
 * These need no GPU (they run on the CPU side of the library). */

const char* qmoe_version(void);
const char* qmoe_last_error(void);

/* generate_dictionary(PairDistribution(p0)).decode_words
 * (dictionary.py:234-279, packed as in :137-147). h_words: uint32[65536*2]. */
int qmoe_generate_decode_words(double p0, uint32_t* h_words);

/* _unpack_all + _build_trie (dictionary.py:150-194): validates the table
 * (pair counts, zero padding, prefix closure, duplicates, single pairs) and
 * fills next_node int32[(65536+1)*9] and entry_of_node int32[65536+1].
 * Returns QMOE_ECORRUPT with qmoe_last_error() naming the failed rule. */
int qmoe_build_trie(const uint32_t* h_words, int32_t* h_next_node, int32_t* h_entry_of_node);

/* --------------------------------------------------------------- dictionary
 * Dictionary upload (Dictionary, dictionary.py:197-224): copies the decode
 * words and the trie to `device` and derives the kernel-private tables
 * (packed <=3-non-zero entry table, length table). Built once per hash. */
int qmoe_dict_create(const uint32_t* h_words, uint64_t hash64, int device, qmoe_dict_t* out);
int qmoe_dict_destroy(qmoe_dict_t dict);
/* max non-zero values per entry, and whether the sparse fast path applies
 * (max_nonzeros <= 3; false e.g. for p0 = 0.7). */
int qmoe_dict_info(qmoe_dict_t dict, uint64_t* hash64, int* max_nonzeros, int* sparse_path);

/* ------------------------------------------------------------------- codec */

/* Row-length check of _decode_range (codec.py:164-169): for every row, the
 * codeword lengths 2*n must sum to cols. d_bad: int32[2] = {number of bad
 * rows, smallest bad row (INT32_MAX if none)}; the caller zeroes it. */
int qmoe_validate_rows(qmoe_dict_t dict, const uint16_t* d_cw, const int32_t* d_row_off,
                       int64_t rows, int64_t cols, int32_t* d_bad, void* stream);

/* decompress (codec.py:175-193 / _decode_range :158-172): d_codes_out is a
 * (rows, cols) uint8 row-major buffer of ternary codes {0,1,2}. Rows that
 * fail the length check are counted in d_bad (as above) and left zero.
 * d_table: NULL (dictionary order) or a frequency codebook (see below). */
int qmoe_decompress(qmoe_dict_t dict, const uint32_t* d_table, const uint16_t* d_cw,
                    const int32_t* d_row_off, int64_t rows, int64_t cols, uint8_t* d_codes_out,
                    int32_t* d_bad, void* stream);

/* fused_matvec (codec.py:209-244) for one matrix and one x vector.
 * d_x: cols values of type x_dtype; d_y: rows float32, updated in place.
 * Rows must have been validated (qmoe_validate_rows): the sparse-path kernel
 * trusts row lengths; d_bad (nullable) is used by the general path. */
int qmoe_fused_matvec(qmoe_dict_t dict, const uint16_t* d_cw, const int32_t* d_row_off,
                      const uint32_t* d_row_minmax, int64_t rows, int64_t cols,
                      const void* d_x, int x_dtype, float* d_y, int32_t* d_bad, void* stream);

/* The same for ntok tokens at once: x is (ntok, ldx), y is (ntok, ldy); each
 * token's result equals qmoe_fused_matvec on that token (decode is shared). */
int qmoe_fused_matmat(qmoe_dict_t dict, const uint16_t* d_cw, const int32_t* d_row_off,
                      const uint32_t* d_row_minmax, int64_t rows, int64_t cols,
                      const void* d_x, int x_dtype, int64_t ntok, int64_t ldx, float* d_y,
                      int64_t ldy, int32_t* d_bad, void* stream);

/* Grouped persistent launch over a device-resident run list: one kernel,
 * one hot-table fill per SM, many (matrix, token) runs. d_n_work = int32[2]
 * {number of runs, total tasks} lives in device memory (written e.g. by
 * qmoe_moe_plan), so the call is graph-capturable with no host
 * synchronisation. max_ntok (<= 2 on the sparse path) bounds work.ntok (sizes
 * the x staging). y_mode: QMOE_Y_ACCUM_F32, QMOE_Y_STORE_F32 or
 * QMOE_Y_RELU_BF16 (fuses the FFN activation into the wi pass epilogue).
 * d_table: entry table the streams are indexed in — NULL for the dictionary's
 * own order, or a codebook from qmoe_codebook_table (streams re-indexed with
 * qmoe_remap; the codebook must map dictionary entry 0 to rank 0). Rows must
 * have been validated (qmoe_validate_rows); d_bad is used by the general
 * (> 3 non-zero) path only. hot_entries: entries of the table staged in
 * shared memory per SM (0 = as many as fit); small launches should stage few.
 * Bits 0-7 of work.lg = lanes per row of the run (log2), bits 8-15 = the
 * checkpoint granularity the matrix stores (0 = same); a run may use any
 * lg <= the stored one (segment boundaries nest). */
int qmoe_grouped_matvec(qmoe_dict_t dict, const uint32_t* d_table, const qmoe_work* d_work,
                        const int32_t* d_n_work, int32_t max_work, int32_t max_cols,
                        int32_t max_ntok, const void* d_x, int x_dtype, int64_t ldx, void* d_y,
                        int y_mode, int64_t ldy, int32_t hot_entries, int32_t* d_bad, void* stream);

/* ------------------------------------------------------- frequency codebook
 * Kernel-private re-indexing of the codeword streams of one model/layer by
 * codeword frequency, so the shared-memory resident prefix of the entry table
 * holds the most used entries (same stream size, decode unchanged):
 *   qmoe_histogram  d_counts[c] += occurrences of c in d_cw[0..n)   (uint32[65536])
 *   qmoe_codebook_table  h_order[k] = codeword of rank k (a permutation of
 *                   0..65535) -> d_table[k] = packed entry of h_order[k]
 *   qmoe_remap      d_out[i] = d_rank_of[d_in[i]] (in place allowed) */
int qmoe_histogram(const uint16_t* d_cw, int64_t n, uint32_t* d_counts, void* stream);
int qmoe_codebook_table(qmoe_dict_t dict, const uint16_t* h_order, uint32_t* d_table);
int qmoe_remap(const uint16_t* d_in, int64_t n, const uint16_t* d_rank_of, uint16_t* d_out,
               void* stream);

/* Row-segment checkpoints for a matrix (kernel-private, derived once): for
 * G = 2^lg (1 <= lg <= 5) segments per row, d_ck[r*(G-1) + j-1] = column where
 * segment j of row r starts. d_table selects the entry order the stream is
 * indexed in (NULL = dictionary). Rows that do not decode to cols values are
 * counted in d_bad (int32[2], as qmoe_validate_rows). */
int qmoe_checkpoints(qmoe_dict_t dict, const uint32_t* d_table, const uint16_t* d_cw,
                     const int32_t* d_row_off, int64_t rows, int64_t cols, int lg, uint16_t* d_ck,
                     int32_t* d_bad, void* stream);

/* Paper Listing 1 kept as the "paper design on B200"
 * baseline: warp per row, lanes 0..27 extract, decode words read through the
 * cache, shuffle reduction. If d_trace is non-NULL it receives, per codeword
 * (stream order), the lane replay of simulate_warp_row (codec.py:293-338):
 * int32[n_cw * 5] = {codeword, pair_count, offset, values of lanes 0..13,
 * values of lanes 14..27} (2 bits per lane, lane i at bits 2*(i % 14)). */
int qmoe_paper_matvec(qmoe_dict_t dict, const uint16_t* d_cw, const int32_t* d_row_off,
                      const uint32_t* d_row_minmax, int64_t rows, int64_t cols,
                      const void* d_x, int x_dtype, float* d_y, int32_t* d_trace,
                      void* stream);

/* encode (codec.py:126-155, _encode_rows :69-123): greedy longest-prefix trie
 * walk, one thread per row. Two phases: count codewords per
 * row into d_counts (int32[rows]), then (after the caller forms
 * row_off = exclusive scan, see qmoe_exclusive_scan) emit the stream. */
int qmoe_encode_count(qmoe_dict_t dict, const uint8_t* d_codes, int64_t rows, int64_t cols,
                      int32_t* d_counts, void* stream);
int qmoe_encode_emit(qmoe_dict_t dict, const uint8_t* d_codes, int64_t rows, int64_t cols,
                     const int32_t* d_row_off, uint16_t* d_cw, void* stream);
/* d_out[0] = 0, d_out[i+1] = sum(d_in[0..i]) for i < n (int32 -> int64 safe
 * accumulation; overflow of int32 is reported via d_out[n] < 0 check). */
int qmoe_exclusive_scan(const int32_t* d_in, int64_t n, int32_t* d_out, void* stream);

/* make_grid + rtn_quantize (quantize.py:91-107, :219-235) for ternary:
 * per-row bf16 (min, max) and nearest-level codes, ties to the smaller
 * magnitude. d_w: float32 (rows, cols). d_minmax_in (nullable) supplies the
 * grid (QuantGrid.minmax_bits); NULL derives it from the row extrema. */
int qmoe_rtn_quantize(const float* d_w, int64_t rows, int64_t cols, const uint32_t* d_minmax_in,
                      uint8_t* d_codes, uint32_t* d_row_minmax, void* stream);

/* ------------------------------------------------------------- MoE dispatch
 * Routed-expert dispatcher (pipeline.py:86-96 gather/scatter order): stable
 * counting sort of the top-1 assignment d_assign[T] into per-expert token
 * lists (d_order, int32[T], expert-major, buffer order within an expert;
 * d_expert_count int32[E]), then the run lists of both FFN passes: one run
 * per (expert, chunk of <= tokens_per_run tokens) covering all rows of
 *   pass 1: wi_e = d_mats[2e]      (d_runs_wi)
 *   pass 2: wo_e = d_mats[2e + 1]  (d_runs_wo)
 * with task0 prefixes filled. d_runs_* hold max_runs (>= T) records;
 * d_n = int32[4] {runs wi, tasks wi, runs wo, tasks wo}. Ids outside
 * [0, E) are dropped (the token gets no expert output). lg_wi / lg_wo: lanes
 * per row (2^lg) of the runs, bounded by each matrix's checkpoint lg; -1 =
 * the matrix's lg. */
int qmoe_moe_plan(const int32_t* d_assign, int32_t T, int32_t E, const qmoe_matrix* d_mats,
                  int32_t tokens_per_run, int32_t lg_wi, int32_t lg_wo, int32_t max_runs, qmoe_work* d_runs_wi,
                  qmoe_work* d_runs_wo, int32_t* d_n, int32_t* d_expert_count, int32_t* d_order,
                  void* stream);

/* One MoE layer step in ONE cooperative persistent launch (the fused form of
 * qmoe_moe_plan + two qmoe_grouped_matvec passes): every CTA rebuilds the
 * dispatcher plan of d_assign[T] in shared memory, runs its share of the wi
 * tasks (h = relu(bf16(wi_e x_t)) stored bf16 in d_h rows of ldh), publishes
 * per-run completion counters, and runs its share of the wo tasks, each wo run
 * waiting only for its own wi run (d_y rows of ldy = bf16(wo_e h_t), f32).
 * Experts: d_mats[2e] = wi_e (d_ff x d_model), d_mats[2e+1] = wo_e, RAW layout;
 * lg_wi / lg_wo <= the checkpoint lg every wi / wo matrix stores.
 * d_counters: int32[2C + 4] for steps of T <= C tokens, zero before the first
 * call except d_counters[2] = C (two parity sets of C per-run counters after
 * a 64-bit arrival ticket; the kernel keeps them consistent across calls with
 * no reset). d_order / d_expert_count (nullable) receive the plan as in
 * qmoe_moe_plan. QMOE_EUNSUPPORTED when E and T do not fit the shared-memory
 * plan (use the grouped path). */
int qmoe_moe_step(qmoe_dict_t dict, const uint32_t* d_table, const int32_t* d_assign, int32_t T,
                  int32_t E, const qmoe_matrix* d_mats, int32_t tokens_per_run, int32_t lg_wi,
                  int32_t lg_wo, int32_t d_model, int32_t d_ff, const void* d_x, int x_dtype,
                  int64_t ldx, uint16_t* d_h, int64_t ldh, float* d_y, int64_t ldy,
                  int32_t* d_counters, int32_t* d_order, int32_t* d_expert_count,
                  int32_t hot_entries, void* stream);

/* qmoe_moe_step plus combine scaling: d_y rows = d_gate[t] * bf16(wo_e h_t)
 * (one f32 multiply after the per-row rounding; d_gate = the router's top-1
 * probability, e.g. from qmoe_route). d_gate == NULL is qmoe_moe_step. The
 * reference has no probability scaling; this is the Switch
 * Transformer combine. */
int qmoe_moe_step_gated(qmoe_dict_t dict, const uint32_t* d_table, const int32_t* d_assign, int32_t T,
                        int32_t E, const qmoe_matrix* d_mats, int32_t tokens_per_run, int32_t lg_wi,
                        int32_t lg_wo, int32_t d_model, int32_t d_ff, const void* d_x, int x_dtype,
                        int64_t ldx, uint16_t* d_h, int64_t ldh, float* d_y, int64_t ldy,
                        int32_t* d_counters, int32_t* d_order, int32_t* d_expert_count,
                        int32_t hot_entries, const float* d_gate, void* stream);

/* One residual MoE block of a model forward in one launch (SURVEY §8 (f),
 * config 5): as qmoe_moe_step_gated on bf16 tokens d_x, but the output is the
 * next layer's input, d_out (bf16, rows of ldo) = bf16(x + gate * bf16(wo_e
 * h_t)) — x's row for tokens without an expert. d_gate nullable (gate 1).
 * d_out must not alias d_x. With d_hash_mult (uint64[d_model], RouterSim's
 * hash multipliers) the block routes its tokens itself with the reference's
 * hash rule (pipeline.py:166-174, bit-exact; d_assign unused, may be NULL;
 * the ids go to d_assign_out when non-NULL): router + block = one launch. */
int qmoe_moe_step_resid(qmoe_dict_t dict, const uint32_t* d_table, const int32_t* d_assign, int32_t T,
                        int32_t E, const qmoe_matrix* d_mats, int32_t tokens_per_run, int32_t lg_wi,
                        int32_t lg_wo, int32_t d_model, int32_t d_ff, const uint16_t* d_x, int64_t ldx,
                        uint16_t* d_h, int64_t ldh, uint16_t* d_out, int64_t ldo, int32_t* d_counters,
                        int32_t hot_entries, const float* d_gate, const uint64_t* d_hash_mult,
                        int32_t* d_assign_out, void* stream);

/* Top-1 router on the device, replaces RouterSim.assign
 * (reference pipeline.py:164-182) for x already in HBM:
 *  QMOE_ROUTE_ARGMAX: scores = f64(x) . proj (d x E row-major f64) + bias
 *    (E f64, nullable), float64 as the reference; d_assign[t] = argmax (lowest
 *    index on ties); d_scores = f64 scratch of qmoe_route_scratch(T, d, E)
 *    elements (its first T * E hold the scores afterwards). Matches the
 *    reference up to near-ties (summation order differs from numpy's matmul).
 *  QMOE_ROUTE_HASH: wrapping-u64 hash of the f32 bit patterns with d_mult[d]
 *    (RouterSim's `mult`), bit-exact; d_proj / d_scores unused.
 * d_gate (f32[T], nullable) receives softmax(scores)[id] (1 for HASH). */
enum { QMOE_ROUTE_ARGMAX = 0, QMOE_ROUTE_HASH = 1 };
int64_t qmoe_route_scratch(int32_t T, int32_t d, int32_t E);
int qmoe_route(int rule, const void* d_x, int x_dtype, int64_t ldx, int32_t T, int32_t d, int32_t E,
               const double* d_proj, const double* d_bias, const uint64_t* d_mult, double* d_scores,
               int32_t* d_assign, float* d_gate, void* stream);

/* Expert-parallel exchange helpers (ep.ExpertParallelMoE):
 * fixed-slot dispatch. Token t with expert id a in [0, E) goes to rank
 * d = a / (E / world), slot d * C + its stable rank among the tokens bound for
 * d (buffer order, pipeline.py:86-90), C = slots_per_rank >= T (the layer's
 * token capacity, equal on every rank): d_slot[t] (-1: no expert),
 * d_id_send[world * C] = rank-local expert id per slot (-1: empty slot),
 * d_send_counts[world] (nullable) = tokens per destination. world <= 64. */
int qmoe_ep_slots(const int32_t* d_assign, int32_t T, int32_t E, int32_t world, int32_t slots_per_rank,
                  int32_t* d_slot, int32_t* d_id_send, int32_t* d_send_counts, void* stream);
/* Row moves by an index (rows of row_bytes, 16-byte aligned): scatter = 1:
 * dst[index[i]] = src[i] (index -1 skipped); scatter = 0: dst[i] =
 * src[index[i]] (index -1: zero row). */
int qmoe_ep_rows(const void* d_src, void* d_dst, int32_t n_rows, int64_t row_bytes, const int32_t* d_index,
                 int scatter, void* stream);
/* Combine gather: d_dst[i][:] (f32, d columns) = f32(d_src_bf16[index[i]][:])
 * (index -1: zero row). Exact for expert outputs (bf16-rounded values), so
 * the combine all-to-all moves bf16 rows. */
int qmoe_ep_combine(const uint16_t* d_src_bf16, float* d_dst, int32_t n_rows, int32_t d, const int32_t* d_index,
                    void* stream);

/* Batched-token decode-then-MMA pass (many tokens per expert, e.g.
 * Switch-large-128 with T in the thousands): for every expert e with tokens
 * d_order[start_e .. start_e + d_expert_count[e]) (qmoe_moe_plan's outputs,
 * start_e = exclusive prefix of the counts), y[t][r] (y_mode as
 * qmoe_grouped_matvec) = bf16(sum_k W_e[r][k] x[t][k]) for all rows r of
 * W_e = d_mats[2e + pass] (RAW layout, rows x cols). x must be bf16
 * (x_dtype QMOE_X_BF16) with ldx % 8 == 0 and a 16-byte aligned base (else
 * QMOE_EINVAL). Each 128-row block of an expert is decoded ONCE per block of
 * tokens_per_block (32 or 64) tokens — a thread per row walks its codewords
 * in order through a ring of two 64-column tiles in shared memory — and
 * multiplied on the tensor cores (tcgen05.mma, bf16 in, fp32 accumulate in
 * TMEM). */
int qmoe_dense_moe_pass(qmoe_dict_t dict, const uint32_t* d_table, const qmoe_matrix* d_mats,
                        int32_t E, int32_t pass, const int32_t* d_expert_count,
                        const int32_t* d_order, int32_t rows, int32_t cols, const void* d_x,
                        int x_dtype, int64_t ldx, void* d_y, int y_mode, int64_t ldy,
                        int32_t tokens_per_block, int32_t hot_entries, void* stream);

/* Debug hook: d_buf = u64[num_sms * 8] receives per-CTA phase stamps of
 * qmoe_moe_step: [0] %globaltimer at the CTA's start, [1..7] SM cycles since
 * then (1 plan done, 2 wi done, 3 wo done, 4-7 plan / window sub-steps);
 * NULL disables. Not for production use. */
int qmoe_debug_step_trace(void* d_buf);
/* Debug hook: an empty kernel of num_sms CTAs x (threads & 0xFFFF) with
 * smem_bytes of dynamic shared memory (launch-floor measurements); threads
 * bits 16+ = launch mode (1 cooperative, 2 programmatic dependent, 3 both). */
int qmoe_debug_empty_launch(int32_t smem_bytes, int32_t threads, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QMOE_H_ */
