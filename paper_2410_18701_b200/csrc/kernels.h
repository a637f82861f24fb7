// kernels.h -- internal launcher interface between the C ABI (baton_api.cu) and
// the sm_100a kernels.  Not part of the public boundary (include/baton.h).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace baton {

constexpr int CHUNK = 256;      // split-K chunk (keys), == BATON_CHUNK
constexpr int MAX_SLOTS = 256;  // per-shard slot limit (kernel-parameter and smem arrays)
constexpr int MAX_SPLICE_JOBS = 64;
constexpr int MAX_MASK_OPS = 2 * MAX_SLOTS + 2;
// split-K partial record: o[D], m, l, 2 pad floats -> 16-B aligned records (float4 I/O)
constexpr int PREC_PAD = 4;

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ------------------------------------------------------------ decode attention
struct DecodeArgs {
    const void *q, *k, *v;
    const void *k_new = nullptr, *v_new = nullptr;   // fused append (a2) when non-null
    int32_t *counters = nullptr;                      // 2 ints after the tickets
    bool dry = false;                                 // only set kernel attributes (pre-capture)
    // the previous launch in the stream was a decode kernel of this shard: the MHA
    // kernel may prefetch before griddepcontrol.wait (decode_attention.cu)
    bool early = false;
    const uint8_t *mask;            // nullable
    const int32_t *lens, *pad;
    void *out;
    float *partial;                 // [slots][q_heads][max_chunks][head_dim + PREC_PAD]: o, m, l, pad
    int32_t *tickets;               // [slots][q_heads] (+2 work counters), zero between calls
    int slots, q_heads, kv_heads, head_dim, max_ctx, max_chunks;
    float scale;
    // decode-step graph, GQA: this launch leaves the split-K merge of its multi-chunk
    // queries to the next launch (no combine kernel in the layer chain), and merges
    // the previous layer's (prev_partial -> prev_out) at its own start, while its first
    // K/V tiles stream in.  The step's last layer is followed by one combine.
    bool defer_merge = false;
    const float *prev_partial = nullptr;
    void *prev_out = nullptr;
};
size_t decode_partial_bytes(int slots, int q_heads, int head_dim, int max_ctx);
size_t decode_ticket_bytes(int slots, int q_heads);
bool decode_supported_head_dim(int head_dim);
cudaError_t launch_decode_attention(const DecodeArgs &a, cudaStream_t s);
// GQA groups of 8 q heads per kv head (head_dim 128): tensor-core variant
bool gqa_supported(int q_heads, int kv_heads, int head_dim);
cudaError_t launch_decode_gqa(const DecodeArgs &a, cudaStream_t s);
// tcgen05 variants: 20 = separate combine kernel, 21 = fused in-kernel merge
cudaError_t launch_decode_gqa_tc(const DecodeArgs &a, cudaStream_t s, bool fused, bool publish = false);
cudaError_t launch_gqa_combine_spin(const DecodeArgs &a, cudaStream_t s);
cudaError_t launch_gqa_combine(const DecodeArgs &a, cudaStream_t s);

// ------------------------------------------------------------ metadata / mask
cudaError_t launch_mask_update(uint8_t *mask, int32_t *S, int32_t *lens, int slots, int max_ctx,
                               cudaStream_t s);
cudaError_t launch_append_kv(void *k_layer, void *v_layer, const void *k_new, const void *v_new,
                             const int32_t *lens, int slots, int kv_heads, int head_dim,
                             int max_ctx, cudaStream_t s);

enum MaskOpKind : int32_t { MOP_ZERO_ROW = 0, MOP_SHIFT_LEFT = 1, MOP_SHIFT_RIGHT = 2, MOP_SET_ROW = 3,
                            MOP_SET_CELL = 4 };
struct MaskOp {
    int32_t kind, slot, a, b;   // ZERO_ROW(slot); SHIFT_LEFT(a=p); SHIFT_RIGHT(a=e); SET_ROW(slot, a=pad, b=S);
                                // SET_CELL(slot, a=column): that one column := 1
};
// Applies `ops` in order to every mask row, then writes S/lens/pad (host values) to the device.
cudaError_t launch_mask_splice(uint8_t *mask, int slots, int max_ctx, const MaskOp *ops, int nops,
                               int32_t *d_S, int32_t *d_lens, int32_t *d_pad, int S,
                               const int32_t *lens, const int32_t *pad, cudaStream_t s);
// Moves mask rows src->dst (dst rows are free), zeroes src, then writes metadata.
cudaError_t launch_mask_move(uint8_t *mask, int slots, int max_ctx, const int32_t *src,
                             const int32_t *dst, int nmoves, int32_t *d_S, int32_t *d_lens,
                             int32_t *d_pad, int S, const int32_t *lens, const int32_t *pad,
                             cudaStream_t s);

// ------------------------------------------------------------ KV splice copies
// For every job, layer l < layers, kv head h < kv_heads and K/V:
//   copy `rows` rows of head_dim bf16 from  src + l*src_ls + h*src_hs
//                                      to   dst + l*dst_ls + h*dst_hs   (strides in elements)
struct CopyJob {
    const void *src_k, *src_v;
    void *dst_k, *dst_v;
    int64_t src_ls, src_hs, dst_ls, dst_hs;
    int32_t rows, pad_;
};
cudaError_t launch_kv_copy(const CopyJob *jobs, int njobs, int layers, int kv_heads, int head_dim,
                           cudaStream_t s);
// NEXT-1: append the W input tokens' K/V of every occupied slot to its cache rows
// [row0[b], row0[b] + W) (row0 < 0: slot skipped), all layers; src token-major
// [layers][slots][W][kv_heads][head_dim].
cudaError_t launch_shape_append(void *k_cache, void *v_cache, const void *k_new, const void *v_new,
                                const int32_t *row0, int layers, int slots, int kv_heads, int head_dim,
                                int max_ctx, int W, cudaStream_t s);

// ------------------------------------------------------------ a8 prefill attention (tcgen05)
bool prefill_supported(int head_dim);
int prefill_varlen_max_prompts();
// n prompts packed along the token axis: Q/O [q_heads][T][D], K/V [kv_heads][T][D],
// prompt i at rows [cu_lens[i], cu_lens[i+1]) (host array), T = cu_lens[n]
cudaError_t launch_prefill_attention_varlen(const void *q, const void *k, const void *v, void *out,
                                            const int32_t *cu_lens, int n, int q_heads, int kv_heads,
                                            int head_dim, float scale, cudaStream_t s);
cudaError_t launch_prefill_attention(const void *q, const void *k, const void *v, void *out, int len,
                                     int q_heads, int kv_heads, int head_dim, float scale,
                                     cudaStream_t s);
// NEXT-1 (vector shaping): attention of the W input tokens of every slot over the
// slot's cache rows [0, lens_b - W + t] where the mask is 1 (prefill_attention.cu).
// q/out: [slots][W][q_heads][128] (token-major); k/v_layer: one layer of the cache;
// lens/pad: the device metadata after the shaped mask update.
cudaError_t launch_extend_attention(const void *q, const void *k_layer, const void *v_layer, void *out,
                                    int W, int slots, int q_heads, int kv_heads, int head_dim, int max_ctx,
                                    const int32_t *lens, const int32_t *pad, const uint8_t *mask,
                                    float scale, cudaStream_t s);

// ------------------------------------------------------------ harness generator
cudaError_t launch_keygen_tokens(void *out, const int32_t *qids, const int32_t *pos, int layers,
                                 int n_slots, int heads, int head_dim, int kind, int layer0,
                                 uint64_t seed, int scale_exp, cudaStream_t s);
cudaError_t launch_keygen_history(void *out, int layers, int heads, int head_dim, int qid,
                                  int pos_begin, int n, int kind, uint64_t seed, int scale_exp,
                                  int64_t head_stride, int64_t layer_stride, cudaStream_t s);

// a8 prefill in the FA4 layout (prefill_fa4.cu): n prompts packed along the token axis
cudaError_t launch_prefill_fa4_varlen(const void *q, const void *k, const void *v, void *out,
                                      const int32_t *cu_lens, int n, int q_heads, int kv_heads,
                                      float scale, float rescale_t, cudaStream_t s);
long long fa4_rescale_count(bool reset);

}  // namespace baton
