/*
 * baton.h -- C ABI of libbaton: the data-parallel hot path of Baton
 * (arXiv 2410.18701, "Baton: Enhancing Batch-wise Inference Efficiency for
 * Large Language Models via Dynamic Re-batching"), B200-native (sm_100a).
 *
 * Citations "P:Lnn" are line numbers of the paper text; "C#" are the
 * readings of ambiguous passages listed in DESIGN.md §3.
 *
 * ------------------------------------------------------------------------
 * Model of the state (§3.1 "Vector Shaping"):
 *   The paper keeps three tensors per batch: input_token, attention_mask and
 *   KV_Cache [layer, 2, batch_size, mul_head, seq_length, embed_length], with a
 *   single shared, growing seq_length S.  Each query b has an `index`
 *   marking where its padding ends: pad_start[b].  Its live length is
 *   lens[b] = S - pad_start[b]; an empty slot has lens 0 (C6).
 *
 *   libbaton keeps the paper's LOGICAL state exactly: S, pad_start[], lens[] and
 *   the 0-1 mask [slots][max_ctx] (logical columns 0..S-1).  The PHYSICAL K/V rows
 *   are slot-relative: the i-th live token of slot b is row i of
 *       K[layer][b][kv_head][0 .. max_ctx)[head_dim]
 *   so logical column j of slot b is physical row j - pad_start[b].  With this
 *   layout the paper's front release and left expansion move
 *   no K/V bytes, and placeholders ("-inf") are never written or read.
 *
 * Conventions (all calls):
 *   - Returns BATON_OK (0) or a negative BATON_E_* code.  Arguments are
 *     validated against the host mirror BEFORE anything is enqueued, so a
 *     failing call leaves host and device state unchanged and needs no sync.
 *   - Device pointers are CALLER-OWNED (e.g. torch tensors); libbaton never
 *     allocates device memory.  Borrowed inputs must stay alive until `stream`
 *     has passed the call.  All work is asynchronous on `stream` (a
 *     cudaStream_t passed as void*; NULL = legacy default stream).
 *   - bf16 = IEEE bfloat16 storage; arithmetic accumulates in fp32; outputs are
 *     rounded to bf16 with round-to-nearest-even (C12, C14).
 *   - A baton_state is used by one host thread and one stream at a time
 *     ("exclusively owned by one decode loop").
 */
#ifndef BATON_H
#define BATON_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BATON_OK            0
#define BATON_E_INVALID    (-1)  /* bad pointer, shape, slot index or argument          */
#define BATON_E_SLOT_BUSY  (-2)  /* insert into an occupied slot                */
#define BATON_E_SLOT_EMPTY (-3)  /* remove / extract of an empty slot           */
#define BATON_E_CAPACITY   (-4)  /* len > max_ctx, S would exceed max_ctx, no room        */
#define BATON_E_CUDA       (-5)  /* a CUDA launch or copy failed (see baton_cuda_error)   */

/* Fixed split-K chunk (keys), relative to each query's live start: results of a
 * query never depend on the batch it sits in (batch invariance). */
#define BATON_CHUNK 256

typedef struct baton_state baton_state;

/* Static shape of one GPU's shard. head_dim in {16, 32, 64, 128};
 * max_ctx (S_cap) a multiple of 16; q_heads a multiple of kv_heads (C11). */
typedef struct {
    int32_t layers, slots, q_heads, kv_heads, head_dim, max_ctx;
} baton_shape;

typedef struct {
    baton_shape shape;
    void    *k_cache;    /* bf16 [layers][slots][kv_heads][max_ctx][head_dim], slot-relative rows */
    void    *v_cache;    /* same layout as k_cache                                              */
    uint8_t *mask;       /* u8 [slots][max_ctx]: the paper's attention_mask, logical columns   */
    void    *workspace;  /* >= baton_workspace_bytes(&shape) bytes, 256-B aligned, any content  */
    size_t   workspace_bytes;
} baton_config;

/* ---------------------------------------------------------------- lifetime */
/* Bytes of a shard's workspace: the device metadata copies, two split-K partial
 * buffers (consecutive layers of baton_decode_step alternate them: a GQA layer's merge
 * runs in the next layer's launch), the tickets / work counters.  Its last
 * baton_decode_workspace_bytes(shape) bytes have the stateless call's layout. */
size_t baton_workspace_bytes(const baton_shape *shape);
/* Bytes of the workspace the stateless baton_decode_attention() needs. */
size_t baton_decode_workspace_bytes(const baton_shape *shape);

/* Creates the host mirror (S = 0, every slot empty) and zero-fills mask and
 * workspace on `stream`.  The caches are not touched (they may hold anything:
 * never-written rows are never read). */
int  baton_create(const baton_config *cfg, void *stream, baton_state **out);
void baton_destroy(baton_state *st);

/* Device copies of the logical metadata kept in the workspace:
 * S (int32[1]), lens (int32[slots]), pad_start (int32[slots]). */
int  baton_device_meta(const baton_state *st, int32_t **S, int32_t **lens, int32_t **pad_start);

/* Host mirror (authoritative, no device sync).  Any out pointer may be NULL.
 * pad_start/lens/occupied are int32[slots]; pad_start of an empty slot is 0. */
int  baton_query(const baton_state *st, int32_t *S, int32_t *pad_start, int32_t *lens,
                 int32_t *occupied);

/* ---------------------------------------------------------------- decode step
 * a1 -- P:L96: "add a column with the value of all 1 to the original
 * attention_mask, indicating that the current input_token is not padding".
 * S += 1; for every occupied slot lens += 1 and mask[b][S-1] = 1; empty slots
 * get mask[b][S-1] = 0 (C6).  Reads/writes the DEVICE copies of S/lens (graph-
 * capturable; the host mirror is advanced identically).
 * Errors: BATON_E_CAPACITY if S+1 > max_ctx. */
int  baton_mask_update(baton_state *st, void *stream);

/* a2 -- P:L96: "appends ... to KV_Cache".  For every occupied slot b and kv head
 * g: K[layer][b][g][lens[b]-1][:] = k_new[b][g][:] (same for V).
 * k_new, v_new: device bf16 [slots][kv_heads][head_dim] (rows of empty slots are
 * ignored).  Call after baton_mask_update.  Bit-exact copy. */
int  baton_append_kv(baton_state *st, int layer, const void *k_new, const void *v_new,
                     void *stream);

/* a3 -- masked scaled-dot-product attention of the decode step (§2.1,
 * P:L52, "based solely on the latest single token").  For every slot b
 * with lens[b] > 0 and q head h (kv head g = h*kv_heads/q_heads, C11):
 *     J   = { j in [0, lens[b]) : mask[b][pad_start[b] + j] == 1 }
 *     s_j = scale * (q[b][h] . K[b][g][j]),   o[b][h] = sum_{j in J} softmax(s)_j V[b][g][j]
 * Masked columns and the placeholders outside [0, lens) are skipped, never
 * loaded into the arithmetic.  Empty slots get a zero output row.
 *   q    : device bf16 [slots][q_heads][head_dim]
 *   k, v : device bf16 [slots][kv_heads][max_ctx][head_dim] of ONE layer
 *   mask : device u8 [slots][max_ctx], or NULL = every column of [0, lens) live
 *   lens, pad_start : device int32 [slots]
 *   out  : device bf16 [slots][q_heads][head_dim]
 *   scale: softmax scale (pass 1/sqrt(head_dim), C10)
 *   workspace: device, >= baton_decode_workspace_bytes(shape) bytes; must be
 *     zero-filled before the first call; every call leaves it reusable.
 * shape->layers is ignored.  A fully masked occupied row is a contract violation
 * and yields a zero output row.  Errors: BATON_E_INVALID. */
int  baton_decode_attention(const void *q, const void *k, const void *v, const uint8_t *mask,
                            const int32_t *lens, const int32_t *pad_start, void *out,
                            const baton_shape *shape, float scale, void *workspace,
                            size_t workspace_bytes, void *stream);

/* a2+a3 on the state's own buffers for one layer: if k_new/v_new are non-NULL
 * the append is performed first (fused launch order), then attention with
 * scale 1/sqrt(head_dim). */
int  baton_decode_layer(baton_state *st, int layer, const void *q, const void *k_new,
                        const void *v_new, void *out, void *stream);

/* One whole decode iteration of the shard: a1 (baton_mask_update), then for every
 * layer l the fused a2+a3 (baton_decode_layer with k_new/v_new).
 *   q, out     : device bf16 [layers][slots][q_heads][head_dim]
 *   k_new,v_new: device bf16 [layers][slots][kv_heads][head_dim]
 * The launch sequence is captured once into a CUDA graph (kernels chained by
 * programmatic dependent launch) and replayed; it is re-captured only when one
 * of the four pointers changes, so keep them fixed (staging buffers).  All
 * kernels read the device copies of S/lens/pad, so the replay needs no host
 * sync.  Errors: BATON_E_INVALID, BATON_E_CAPACITY (S+1 > max_ctx). */
int  baton_decode_step(baton_state *st, const void *q, const void *k_new, const void *v_new,
                       void *out, void *stream);

/* ---------------------------------------------------------------- KV splice
 * a4 -- P:L105 "set all the values of the query^2 part of the current
 * attention_mask tensor to 0", then P:L123-124 resource releasing: the
 * [0 : min(index_i)] front segment of KV_Cache and attention_mask is released
 * (min over occupied slots; everything if none, C5).
 * slots: HOST int32[n], each occupied, no duplicates.  The K/V rows are left in
 * place as inert placeholders; zero K/V bytes move.  *released (nullable, host)
 * receives p.  Errors: BATON_E_INVALID, BATON_E_SLOT_EMPTY. */
int  baton_remove(baton_state *st, const int32_t *slots, int n, int32_t *released, void *stream);

/* a5 -- P:L132-138 vector embedding of a prefilled query into empty `slot`:
 *   len <= S: end-aligned, pad_start[slot] = S - len, mask row 0^{S-len} 1^{len}
 *   len >  S: expand on the left by e = len - S: every other row's mask shifts
 *             right by e with 0 fill and its pad_start grows by e; S = len;
 *             pad_start[slot] = 0, mask row all 1.
 * Then K[l][slot][g][0:len] = k_pref[l][g][0:len] for every layer/kv head (same
 * for V).  k_pref, v_pref: device bf16 [layers][kv_heads][len][head_dim],
 * contiguous.  Errors: BATON_E_SLOT_BUSY, BATON_E_CAPACITY (len < 1 or > max_ctx),
 * BATON_E_INVALID. */
int  baton_insert(baton_state *st, int slot, const void *k_pref, const void *v_pref, int len,
                  void *stream);

/* a5 batched: the n inserts of one iteration in ONE splice launch (plus one
 * metadata launch).  Same result as n baton_insert calls in array order (C7).
 * slots, lens: HOST int32[n]; k_pref, v_pref: HOST arrays of n device pointers. */
int  baton_insert_many(baton_state *st, int n, const int32_t *slots, const void *const *k_pref,
                       const void *const *v_pref, const int32_t *lens, void *stream);

/* a6 -- P:L144 "temporarily store the Keys and Values" of an occupied slot:
 * k_out[l][g][0:lens] = K[l][slot][g][0:lens] (its live region, C16), same for V.
 * k_out, v_out: device (or cudaHostRegister'ed/pinned host) bf16
 * [layers][kv_heads][lens[slot]][head_dim].  Metadata is unchanged; call
 * baton_remove afterwards to free the slot.  Errors: BATON_E_SLOT_EMPTY. */
int  baton_extract(baton_state *st, int slot, void *k_out, void *v_out, void *stream);

/* a7 -- P:L147 batch-size scaling: move every occupied slot with index >=
 * n_active into the lowest free slot < n_active, ascending (C19); copies their
 * live K/V rows, mask rows and metadata.  old_to_new (HOST int32[slots], nullable)
 * receives the permutation (identity for unmoved slots).
 * Errors: BATON_E_CAPACITY if the occupied slots do not fit. */
int  baton_compact(baton_state *st, int n_active, int32_t *old_to_new, void *stream);

/* ---------------------------------------------------------------- prefill side
 * a8 -- P:L132 "all original queries awaiting processing are initially
 * prefilled by the model", decoupled from decoding (P&D, P:L215 asynchronous).
 * Causal scaled-dot-product attention of a new query over its own prompt:
 *     O[h][i] = sum_{j <= i} softmax_j(scale * Q[h][i] . K[g][j]) V[g][j],
 * g = h*kv_heads/q_heads (C11), i.e. for every i the decode attention (a3) of
 * the prefix [0, i].  Runs on the tensor cores (tcgen05.mma, TMEM accumulators,
 * TMA tiles); P is rounded to bf16 for the P.V product.
 *   Q, O : device bf16 [q_heads][len][head_dim];  K, V : [kv_heads][len][head_dim]
 *          (one layer of the prefilled K/V that baton_insert embeds)
 *   head_dim must be 128; 16-B aligned pointers.  Run it on a side stream to
 *   overlap the decode loop (the insert then waits on an event).
 * Errors: BATON_E_INVALID. */
int  baton_prefill_attention(const void *q, const void *k, const void *v, void *out, int len,
                             const baton_shape *shape, float scale, void *stream);

/* a8, batched (NEXT-2: the prefill side of P&D at scale): the same causal
 * attention for n prompts in ONE launch, e.g. every query queued for insertion in an
 * iteration ("all original queries awaiting processing are initially
 * prefilled"; P:L215 asynchronous P&D).  Prompt i is its own causal problem; no
 * attention crosses prompts.
 *   Q, O : device bf16 [q_heads][T][head_dim];  K, V : [kv_heads][T][head_dim], the
 *          prompts packed along the token axis: prompt i occupies rows
 *          [cu_lens[i], cu_lens[i+1]), T = cu_lens[n].
 *   cu_lens : HOST int32 [n+1], cu_lens[0] = 0, strictly increasing (every prompt
 *          has >= 1 token); read during the call only.
 *   1 <= n <= 64 and sum_i ceil(len_i / 128) <= 1024.  Same result, row for row and
 *   bit for bit, as n separate baton_prefill_attention calls.
 * Errors: BATON_E_INVALID. */
int  baton_prefill_attention_varlen(const void *q, const void *k, const void *v, void *out,
                                    const int32_t *cu_lens, int n, const baton_shape *shape,
                                    float scale, void *stream);

/* ---------------------------------------------------------------- NEXT-1
 * The vector-SHAPING iteration: Baton WITHOUT P&D decoupling (the
 * "Ours" column of the paper's Table 2 ablation).  Raw queries join the
 * batch with their whole prompt; "to align the dimensions of IT, it is necessary
 * to pad the latest token of query^0 and query^1 to the same length as query^3"
 * (P:L103).  One call = one iteration of input width W over all layers:
 *   - every occupied slot (survivor) inputs its decode token at t = 0 and W-1
 *     padding tokens: mask columns [S, S+W) := 1 0^(W-1) ("appended with values
 *     of 0 according to the padding"), lens += W;
 *   - every new slot (must be empty, i.e. removed: its row is already zero)
 *     inputs its prompt, l = new_lens[i] <= W tokens: mask row := 0^S 1^l 0^(W-l),
 *     pad = S (its live region starts here), lens = W;
 *   - S += W (reading C4: mask and KV both grow by the input width);
 *   - K/V rows [lens_before, lens_before + W) of each slot := k_new/v_new rows;
 *   - for every slot and input token t: attention over the slot's cache rows
 *     r <= (lens_before + t) with mask 1 (causal inside the new block), on the
 *     tensor cores (the a8 kernel with a per-slot prefix and the mask).  Rows of
 *     padding tokens are computed too: that is the bubble the paper measures
 *     ("even other queries that are already in the decoding phase will
 *     also have the same overhead").
 *   W >= max(1, max new_lens); head_dim must be 128.
 *   new_slots, new_lens : HOST int32[n_new]
 *   q, out       : device bf16 [layers][slots][W][q_heads][head_dim] (token-major,
 *                  as a model's QKV projection produces them)
 *   k_new, v_new : device bf16 [layers][slots][W][kv_heads][head_dim]; rows of
 *                  padding tokens are stored (masked) and must be finite
 *   Empty slots produce zero output rows.  Host mirror and device metadata are
 *   updated like a1 (no baton_mask_update for this iteration).
 * Errors: BATON_E_INVALID, BATON_E_SLOT_BUSY (a new slot is occupied),
 *         BATON_E_CAPACITY (new_lens out of [1, W], or S + W > max_ctx). */
int  baton_shape_step(baton_state *st, int W, int n_new, const int32_t *new_slots,
                      const int32_t *new_lens, const void *q, const void *k_new, const void *v_new,
                      void *out, void *stream);

/* ---------------------------------------------------------------- misc */
const char *baton_error_string(int code);
/* The cudaError_t of the last BATON_E_CUDA returned on this thread. */
int  baton_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BATON_H */
