/*
 * cce_b200.h — C ABI of libcce_b200.so, the B200 (sm_100a) Cut Cross-Entropy hot path.
 *
 * The reference (arxiv 2411.09009, /root/reference/pkg/src/cce) is a pure-Python package whose
 * hot path is three functions composed by cce_loss.  Each entry point below replaces one of
 * them; the Python layer (paper_2411_09009_b200/api.py) binds this header with ctypes exactly
 * as a reference-side maintainer would.
 *
 * Conventions
 *  - Every function returns 0 on success, nonzero on failure; cce_last_error() then describes it.
 *    No C++ exception crosses the ABI.  No host synchronisation is performed.
 *  - Pointers are device pointers unless stated; `stream` is a cudaStream_t (void*).
 *  - E is bf16 [n, d] row-major, C is bf16 [v, d] row-major (reference core.py:5-8 layout:
 *    token-major embeddings, vocab-major classifier).  d must be a multiple of 8.
 *  - Outputs and workspaces are caller-allocated (so torch's allocator accounts every byte,
 *    mirroring instrument.py's scratch/output split).
 */
#ifndef CCE_B200_H
#define CCE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Message of the last failing call on this thread. */
const char* cce_last_error(void);
int cce_abi_version(void);
/* Kernels launched by this library so far (all threads; CUB's sort kernels not included). */
unsigned long long cce_launch_count(void);

/* ---- forward: indexed_matmul (kernels.py:204-251) + lse_forward (kernels.py:254-319) ----
 * One fused persistent tcgen05 kernel: per token row, the log-sum-exp over this shard's
 * vocabulary rows [vocab_start, vocab_start + v) (lse_local) and the target logit when the
 * target falls in the shard (correct, else 0).  softcap > 0 applies cap*tanh(z/cap) to every
 * logit.  Logits never reach HBM; ws holds splits*n float2 partials. */
size_t cce_fwd_workspace_bytes(int64_t n, int64_t d, int64_t v);
int cce_fwd(const void* E, const void* C, const int64_t* targets, int64_t n, int64_t d, int64_t v,
            int64_t ignore_index, int64_t vocab_start, float softcap, void* ws, size_t ws_bytes,
            float* lse_local, float* correct, void* stream);

/* ---- combine shards (log_add_exp merge, kernels.py:121-137; scatter kernels.py:539-547) ----
 * lse_parts / correct_parts are [num_shards][n]; lse_out = log-add-exp over shards (0 at
 * ignored rows), loss_out = lse - sum(correct) (0 at ignored rows). */
int cce_merge_shards(int num_shards, const float* lse_parts, const float* correct_parts,
                     const int64_t* targets, int64_t ignore_index, int64_t n, float* lse_out,
                     float* loss_out, void* stream);
/* The same, plus the reference's label-range check (check_vocab, core.py:110-114) without a
 * host read: with v_total > 0 a row whose target is neither ignore_index nor in [0, v_total) gets
 * a NaN loss and *label_error is set to 1 (sticky; the caller reads it asynchronously and raises
 * the reference's ValueError at its next call).  label_error may be NULL. */
int cce_merge_shards_checked(int num_shards, const float* lse_parts, const float* correct_parts,
                             const int64_t* targets, int64_t ignore_index, int64_t n, int64_t v_total,
                             int* label_error, float* lse_out, float* loss_out, void* stream);

/* ---- vocabulary order (compute_vocab_order, kernels.py:145-160) ----
 * cce_ebar: column sums of the rows of E whose target != ignore_index (targets may be NULL =
 * all rows), summed in a fixed order (bit-reproducible) through a workspace of
 * cce_ebar_workspace_bytes.  cce_vocab_order: key = C . ebar_sum / n_valid (the reference's
 * mean_logits), perm = stable descending argsort of key (ties by ascending index); n_valid is a
 * device int. */
size_t cce_ebar_workspace_bytes(int64_t n, int64_t d);
int cce_ebar(const void* E, const int64_t* targets, int64_t ignore_index, int64_t n, int64_t d,
             float* ebar_sum, void* ws, size_t ws_bytes, void* stream);
size_t cce_sort_workspace_bytes(int64_t v);
int cce_vocab_order(const void* C, const float* ebar_sum, const int* n_valid, int64_t v, int64_t d,
                    int32_t* perm, float* key_out, void* ws, size_t ws_bytes, void* stream);

/* ---- backward (lse_backward, kernels.py:327-486) ----
 * cce_compact_rows: filter_ignored (kernels.py:494-510) on the device: row_map[k] = k-th row
 * whose target != ignore_index (row_map sized ceil(n/128)*128, tail zero), *n_valid = count.
 * Nothing is read back to the host.
 * cce_bwd_prep: perm padded to a multiple of 256 and its inverse, and per ORIGINAL row the label
 * position in tile order (-1 = ignored or owned by another shard).  perm may be NULL.
 *
 * cce_bwd: rows are the compacted rows (row_map, *n_valid); E is compacted into the workspace
 * (or, with e_gather, read through row_map by TMA gather4).  C is either the classifier in
 * natural order (perm_padded NULL), sorted rows gathered on the fly (perm_padded, c_sorted = 0)
 * or the pre-sorted C[perm] (c_sorted = 1, see cce_gather_rows).  Token tiles are processed in
 * groups of `group_tiles`; kept tiles take compact 64 KiB bf16 S-hat slots, `capacity_tiles` of
 * them.  Per group: (B1) recompute every 128x256 logit tile on the tensor cores and keep it iff
 * it holds a label or some S = exp(z - lse) >= eps (block_skip_decision, kernels.py:140-142;
 * label tiles exempt as in kernels.py:447-455; eps = 0 disables filtering; token tiles whose
 * upstream is all zero are skipped, kernels.py:434-438), storing S-hat = up * (S - onehot);
 * (B2) dE[n] = sum_m S-hat[n,m] C[m] and (B3) dC[m] (+)= sum_n S-hat[n,m]^T E[n], both
 * output-stationary in TMEM, no atomics.  lse / upstream / pos are indexed by original row.
 * de_out: [n, d] bf16 (or fp32 if de_fp32), written for every compact row; the caller zeroes it.
 * dc: [v, d] bf16, fully written.  counters[3] += {kept, eps-skipped, zero-upstream-skipped}
 * (BackwardStats, kernels.py:66-76).  If a group keeps more tiles than the capacity, *overflow
 * is set and the outputs are invalid; a second call with run_if = overflow and
 * capacity_tiles >= group_tiles * ceil(v/256) then recomputes them (every kernel of a call with
 * *run_if == 0 exits immediately, so the fallback needs no host synchronisation). */
int cce_compact_rows(const int64_t* targets, int64_t ignore_index, int64_t n, int32_t* row_map,
                     int* n_valid, void* stream);
int cce_bwd_prep(const int32_t* perm, int64_t v, const int64_t* targets, int64_t ignore_index,
                 int64_t vocab_start, int64_t n, int32_t* perm_padded, int32_t* inv_perm, int32_t* pos,
                 void* stream);
size_t cce_bwd_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t group_tiles,
                               int64_t capacity_tiles);
int cce_bwd(const void* E, const void* C, const int32_t* perm_padded, int c_sorted,
            const int32_t* row_map, const int* n_valid, const int32_t* pos, const float* lse,
            const float* upstream, int64_t n, int64_t d, int64_t v, float softcap, float eps,
            int64_t group_tiles, int64_t capacity_tiles, const int* run_if, int e_gather, void* ws,
            size_t ws_bytes, void* de_out, int de_fp32, void* dc, unsigned long long* counters,
            int* overflow, void* stream);

/* ---- filter decision taken from the forward (the default training path) ----
 * The reference decides per (token block, vocab block) tile whether lse_backward recomputes it
 * (kernels.py:434-455).  Here the forward already visits every tile, so it records each row's
 * max raw logit per tile and the backward recomputes only the kept tiles.
 *
 * cce_fwd_tiles: forward over the COMPACTED rows E_c (row k = E[row_map[k]], k < *n_valid; see
 * cce_compact_rows / cce_gather_rows) against the classifier in tile order C_t (C[perm] with
 * vocab sorting, else C).  pos[i] (per ORIGINAL row, cce_bwd_prep) is the label position in tile
 * order or -1.  lse_local / correct are per ORIGINAL row (undefined / 0 at ignored rows).
 * tile_max: [ceil(n/128)][ceil(v/256)][128] fp32 (cce_tile_max_bytes), the max raw logit of
 * each compact row in each tile.  ws as cce_fwd (cce_fwd_workspace_bytes).
 * Label tiles (optional, lab_buf != NULL): a tile holding some row's label is always kept by the
 * backward (kernels.py:447-455), so the forward stores it -- fp16 of z' - z'max(row), <= 0 and
 * exact near the row max -- in one of lab_capacity 64 KiB slots of lab_buf; lab_slot
 * [ceil(n/128)][ceil(v/256)] (-1 = none) and lab_list [lab_capacity] (token tile, vocab tile) int2
 * map them, *lab_count counts the slots handed out (tiles past the capacity are simply
 * recomputed).  lab_buf is the head of the S-hat buffer later passed to cce_bwd_kept.
 *
 * cce_bwd_kept: the backward from tile_max.  Keeps tile (n, m) iff its upstream is not all zero
 * and it holds a label or some S >= eps (the same strict test as cce_bwd, eps > 0 required);
 * kept tiles stored by the forward become S-hat in place, the other kept tiles are recomputed,
 * then the dE / dC passes of cce_bwd.  shat: [lab_capacity + capacity_tiles][128][256] bf16, the
 * label region first (lab_slot / lab_list / lab_count from cce_fwd_tiles, or lab_slot NULL: none).
 * stats (optional, 2 ints): label tiles stored, tiles the whole-batch pass recomputes (sizing
 * hints for the next call).  dC rows land
 * through perm_padded (NULL = tile order is C's order).  capacity_tiles >= ceil(v/256) S-hat
 * slots: if the whole batch keeps more tiles than that, *overflow = 1, the whole-batch pass is
 * skipped on the device and token-tile groups sized for the worst case run instead (each kernel
 * gated on *overflow; dC accumulated in bf16 after the first group) -- no host synchronisation.
 * counters as cce_bwd.
 * de_done_event (a cudaEvent_t, may be NULL) is recorded on the stream once every dE write of the
 * call has been enqueued, before the dC pass: a vocab-parallel caller all-reduces dE on another
 * stream while dC runs.
 * dc may alias C_t (dc == C_t): the sorted copy is last read by the dE pass, so its storage can
 * become the dC output and no transient holds a second V x D matrix.  C is then the caller's
 * classifier in its own row order and the fallback groups read it through perm_padded (row
 * gathers) instead of C_t, which an earlier group's dC pass has overwritten.  C may be NULL when
 * dc does not alias C_t.
 * Vocabulary groups (cce_fwd_tiles and cce_bwd_kept): C_t may hold only the sorted rows
 * [pos_offset, pos_offset + v) of the vocabulary, pos_offset a multiple of 256; label positions
 * pos are global and pos - pos_offset is group-local, tile_max is the group's own
 * [ceil(n/128)][ceil(v/256)][128] block and perm_padded points at the group's first entry.  With
 * de_accumulate (fp32 dE only) the call adds its dE into de_out instead of writing it, so the
 * groups of one backward accumulate in a fixed order.
 * de_out or dc may be NULL (not both): that pass is skipped (an input that needs no gradient,
 * e.g. a frozen classifier).  kept_per_vtile (optional, ceil(v/256) ints) receives the number of
 * kept tiles of each vocab tile (sizing hints: low_memory groups follow the vocabulary's
 * kept density). */
size_t cce_tile_max_bytes(int64_t n, int64_t v);
int cce_fwd_tiles(const void* E_c, const void* C_t, const int32_t* row_map, const int* n_valid,
                  const int32_t* pos, int64_t pos_offset, int64_t n, int64_t d, int64_t v, float softcap, void* ws,
                  size_t ws_bytes, float* lse_local, float* correct, float* tile_max, void* lab_buf,
                  int64_t lab_capacity, int32_t* lab_slot, void* lab_list, int* lab_count, void* stream);
/* cce_fwd_gather: cce_fwd_tiles without copies -- E is the caller's [n][d] embeddings (rows read
 * through row_map unless it is the identity) and C the caller's classifier in its own row order,
 * read through perm_padded (cce_bwd_prep) with cp.async row gathers, so neither the compacted E
 * nor the sorted classifier exists.  No label-tile store.  Results are bit-identical to
 * cce_fwd_tiles on the copies. */
int cce_fwd_gather(const void* E, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                   const int* n_valid, const int32_t* pos, int64_t pos_offset, int64_t n, int64_t d, int64_t v,
                   float softcap, void* ws, size_t ws_bytes, float* lse_local, float* correct, float* tile_max,
                   void* stream);
size_t cce_bwd_kept_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t capacity_tiles,
                                    int64_t lab_capacity);
int cce_bwd_kept(const void* E_c, const void* C_t, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                 const int* n_valid, const int32_t* pos, int64_t pos_offset, const float* lse, const float* upstream,
                 const float* tile_max, int64_t n, int64_t d, int64_t v, float softcap, float eps,
                 int label_split, void* shat, int64_t lab_capacity, const int32_t* lab_slot,
                 const void* lab_list, const int* lab_count, int64_t capacity_tiles, void* ws, size_t ws_bytes,
                 void* de_out, int de_fp32, int de_accumulate, void* dc, unsigned long long* counters,
                 int* overflow, int* stats, int* kept_per_vtile, void* de_done_event, void* stream);

/* ---- low-memory backward: vocabulary groups (low_memory=True) ----
 * lse_backward over groups of `group_vtiles` vocab tiles in tile order: per group, the group's
 * classifier rows (C[perm] slice gathered into the workspace, or a view of C when perm_padded is
 * NULL), the filter pass over every (token tile, group vocab tile) with S-hat slots for the
 * worst case (ceil(n/128) * group_vtiles), dE accumulated into the caller-zeroed fp32 de_f32
 * (fixed group order), and dC of the group's vocab tiles written once.  Transient memory:
 * compacted E + one group's classifier rows + the group's S-hat slots + maps
 * (cce_bwd_lowmem_workspace_bytes); no allocation grows with the kept-tile count.  Rows are the
 * compacted rows (row_map, *n_valid); pos / lse / upstream per original row (cce_bwd_prep). */
size_t cce_bwd_lowmem_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t group_vtiles);
int cce_bwd_lowmem(const void* E, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                   const int* n_valid, const int32_t* pos, const float* lse, const float* upstream,
                   int64_t n, int64_t d, int64_t v, float softcap, float eps, int label_split,
                   int64_t group_vtiles, void* ws, size_t ws_bytes, float* de_f32, void* dc,
                   unsigned long long* counters, void* stream);

/* cce_fwd_group: cce_fwd_tiles over one vocabulary group of the sorted order (the bounded-memory
 * training forward).  C_g holds the group's sorted rows [v0, v0 + v_group) (v0 a multiple of 256),
 * label positions pos are global (pos - v0 is group-local); lse_part / correct_part are the group's
 * partials (merge with cce_merge_shards); tile_max is the GLOBAL [ceil(n/128)][ceil(v_total/256)]
 * [128] array, the group writing its own vocab tiles.  E is the caller's E with e_gather = 1 (rows
 * read through row_map unless the compaction is the identity) or a compacted copy (e_gather = 0). */
int cce_fwd_group(const void* E, int e_gather, const void* C_g, const int32_t* row_map, const int* n_valid,
                  const int32_t* pos, int64_t v0, int64_t n, int64_t d, int64_t v_group, int64_t v_total, float softcap,
                  void* ws, size_t ws_bytes, float* lse_part, float* correct_part, float* tile_max, void* stream);
/* cce_fwd_group for the groups of one sweep: flags bit 0 = correct_part already zeroed (a label lands
 * in exactly one group, so every group may write one shared array), bit 1 = leave the group's
 * (max, sum-exp) partials ([cce_fwd_splits(n, d, v_group)][n] float2, log2 units) in ws and skip
 * lse_part; cce_combine_parts then finishes lse over the groups' partials ([count][n] float2) at
 * once, or, with lse_out == NULL, folds them into parts[0] (a running partial). */
int cce_fwd_group_ex(const void* E, int e_gather, const void* C_g, const int32_t* row_map, const int* n_valid,
                     const int32_t* pos, int64_t v0, int64_t n, int64_t d, int64_t v_group, int64_t v_total,
                     float softcap, void* ws, size_t ws_bytes, float* lse_part, float* correct_part, float* tile_max,
                     int flags, void* stream);
/* One launch of the bounded forward's group chain (ops.forward_stream; replaces the per-group
 * gather launches and stream waits around cce_fwd_group_ex): sweeps group g from its buffer C_g
 * once *ready >= 1 (nullptr: stream order), without waiting for the previous launch to finish
 * (no_dep_wait); counts its exited CTAs in *exit_ctr, the last setting *released = 1; and, in the
 * same launch, gathers the next group's rows C[next_perm[r]] (r < next_rows) into next_dst once
 * *next_wait >= 1 (the launch before this one has exited; nullptr: at once), counting shares in
 * *next_ctr, the last setting *next_done = 1 (the next launch's `ready`).  next_dst NULL: no
 * gather.  Counters and flags start at zero. */
int cce_fwd_group_sync(const void* E, int e_gather, const void* C_g, const int32_t* row_map, const int* n_valid,
                       const int32_t* pos, int64_t v0, int64_t n, int64_t d, int64_t v_group, int64_t v_total,
                       float softcap, void* ws, size_t ws_bytes, float* correct_part, float* tile_max,
                       const int* ready, int* exit_ctr, int* released, int no_dep_wait, const void* C,
                       const int32_t* next_perm, int64_t next_rows, void* next_dst, const int* next_wait,
                       int* next_ctr, int* next_done, void* stream);
int cce_fwd_splits(int64_t n, int64_t d, int64_t v);
int cce_combine_parts(const void* parts, int count, int64_t n, float* lse_out, void* stream);

/* ---- streamed backward: transient memory independent of the kept-tile count ----
 * cce_bwd_stream replaces lse_backward (kernels.py:327-486) on the training path.  The decision
 * comes from the forward's tile maxima (tile_max [ceil(n/128)][ceil(v/256)][128], the layout of
 * cce_fwd_tiles / cce_fwd_group), exactly as in cce_bwd_kept.  Every kept tile is then recomputed
 * once, in vocabulary-tile-major order, by the recomputing CTAs of one persistent kernel and
 * streamed to its dC and dE CTAs through `ring` ([ring_slots][128][256] bf16; 512 slots = 32 MiB;
 * ops.stream_ring_slots uses 8 per token tile above 64 token tiles, up to 2048); no S-hat buffer
 * grows with the kept count.  At most 2048 token tiles per call (larger batches: token chunks
 * with cce_bwd_stream_ex).
 *   E          rows of the token tiles: the caller's E with e_gather = 1 (rows are read through
 *              row_map unless the compaction is the identity) or a compacted copy with e_gather = 0
 *   C          the caller's classifier; with a vocabulary order (perm_padded / inv_perm from
 *              cce_bwd_prep) its rows are gathered into c_sorted ([v][d] bf16).  c_sorted may be dc:
 *              dC is then written in the sorted order over the sorted copy and moved back to
 *              vocabulary order in place (no second V x D buffer)
 *   de_out     [n][d] bf16 (or fp32 with de_fp32), rows of ignored tokens left untouched (zero them)
 *   counters   [3] u64 += {kept, eps-skipped, zero-upstream-skipped} (BackwardStats)
 * de_done_event (optional) is recorded once every dE write is enqueued.  ring_slots >= 64. */
size_t cce_bwd_stream_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t ring_slots);
/* diagnostics: byte offsets of the stream lists inside the workspace (13 values; see
 * scripts/stream_lists_check.py), returns the window size in items */
int cce_bwd_stream_debug_layout(int64_t n, int64_t d, int64_t v, int64_t ring_slots, int64_t* offsets);
int cce_bwd_stream(const void* E, int e_gather, const void* C, void* c_sorted, const int32_t* perm_padded,
                   const int32_t* inv_perm, const int32_t* row_map, const int* n_valid, const int32_t* pos,
                   const float* lse, const float* upstream, const float* tile_max, int64_t n, int64_t d, int64_t v,
                   float softcap, float eps, int label_split, void* ring, int64_t ring_slots, void* ws,
                   size_t ws_bytes, void* de_out, int de_fp32, void* dc, unsigned long long* counters,
                   void* de_done_event, void* stream);

/* cce_bwd_stream with flags: bit 0 = c_sorted already holds C[perm] (no gather), bit 1 = add dC
 * into dc (vocabulary order, bf16 accumulate; dc must not be c_sorted).  Token chunks of a large
 * batch run one call each over a shared sorted copy (ops.backward_from_stream_state). */
int cce_bwd_stream_ex(const void* E, int e_gather, const void* C, void* c_sorted, const int32_t* perm_padded,
                      const int32_t* inv_perm, const int32_t* row_map, const int* n_valid, const int32_t* pos,
                      const float* lse, const float* upstream, const float* tile_max, int64_t n, int64_t d,
                      int64_t v, float softcap, float eps, int label_split, void* ring, int64_t ring_slots, void* ws,
                      size_t ws_bytes, void* de_out, int de_fp32, void* dc, unsigned long long* counters,
                      void* de_done_event, int flags, void* stream);

/* diagnostics / tests: the in-place row unpermutation the streamed backward applies to dC when it
 * lands in the sorted order: X[perm[p]] <- X[p] for p < v, X bf16 [v][d] (d % 8 == 0), inv the
 * inverse permutation; ws of cce_bwd_stream_workspace_bytes(1, d, v, 512) bytes */
int cce_unpermute_rows(void* X, const int32_t* perm, const int32_t* inv, int64_t v, int64_t d, void* ws,
                       size_t ws_bytes, void* stream);

/* ---- paper ordering (label_split = 1 in cce_bwd_kept / cce_bwd_lowmem) ----
 * PAPER.md Alg. 3 filters tiles on S alone, before the one-hot subtraction;
 * the reference instead never skips a tile holding a label (kernels.py:447-455).
 * With label_split = 1 the decision ignores labels and S-hat carries no -1; cce_label_terms then
 * applies the label term exactly, as the backward of the indexed matmul:
 *   dE[i] += coef_i C[x_i],  dC[x_i] += sum_{i: x_i} coef_i E[i],  coef_i = -up_i (1 - tanh^2)
 * with tanh = correct_i / softcap (correct = the forward's per-row target logit; 1 without
 * softcap).  E / C are the ORIGINAL matrices, perm_padded maps tile order to C rows (or NULL);
 * de is bf16 or fp32 (de_fp32) per original row; dC gets one bf16 rounding per labelled row.
 * Tokens sharing a label are summed in a fixed order (deterministic). */
size_t cce_label_terms_workspace_bytes(int64_t n);
int cce_label_terms(const void* E, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                    const int* n_valid, const int32_t* pos, const float* upstream, const float* correct,
                    int64_t n, int64_t d, int64_t v, float softcap, void* ws, size_t ws_bytes, void* de,
                    int de_fp32, void* dc, void* stream);

/* ---- reductions (default_upstream, core.py:181-200; linear_cross_entropy's reduction) ----
 * reduction: 0 none, 1 sum, 2 mean over valid rows (an all-ignored batch gives 0, not NaN).
 * cce_reduce_loss: *out = sum of the per-row losses (or that / n_valid); one block, fixed order.
 * cce_upstream: up[i] = 0 at ignored rows, else grad[i] (none, grad is [n]) or grad[0] (sum) or
 * grad[0] / n_valid (mean).  Device scalars throughout: no host synchronisation. */
int cce_reduce_loss(const float* loss, const int64_t* targets, int64_t ignore_index, int64_t n,
                    int reduction, float* out, void* stream);
int cce_upstream(const float* grad, const int64_t* targets, int64_t ignore_index, int64_t n, int reduction,
                 float* up, void* stream);

/* dst[i] = src[index[i]] for bf16 rows of `cols` elements: materialises the vocabulary-sorted
 * classifier C[perm] so the backward loads plain tiles (c_sorted = 1). */
int cce_gather_rows(const void* src, const int32_t* index, int64_t rows, int64_t cols, void* dst,
                    void* stream);

/* fp32 -> bf16 cast of the dE accumulator (count % 4 == 0). */
int cce_f32_to_bf16(const float* x, void* y, int64_t count, void* stream);

/* indexed_matmul alone (kernels.py:204-251): out[i] = C[x_i - vocab_start] . E[i], 0 when the
 * target is ignored or outside the shard; softcap applied when > 0. */
int cce_indexed_dot(const void* E, const void* C, const int64_t* targets, int64_t n, int64_t d,
                    int64_t v, int64_t ignore_index, int64_t vocab_start, float softcap, float* out,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CCE_B200_H */
