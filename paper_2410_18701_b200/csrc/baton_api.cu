// baton_api.cu -- the C ABI of libbaton (include/baton.h, include/baton_keygen.h):
// argument validation against the host mirror of the logical state, then
// asynchronous launches on the caller's stream.  The host mirror follows the
// paper's state machine (P:L96 step, P:L105 remove, P:L124 release, P:L137
// embedding, P:L144 store, P:L147 scaling) on metadata only; every byte of
// device data is touched by the kernels in decode_attention.cu / meta.cu /
// splice.cu.
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include <cuda_bf16.h>

#include "../../include/baton.h"
#include "../../include/baton_keygen.h"
#include "kernels.h"

using namespace baton;

struct baton_state {
    baton_config cfg;
    baton_shape sh;
    int S = 0;
    std::vector<int32_t> pad, lens, occ;
    int32_t *d_S = nullptr, *d_lens = nullptr, *d_pad = nullptr;
    int32_t *tickets = nullptr;
    float *partial = nullptr;
    float *partial2 = nullptr;    // the decode step's second split-K buffer (deferred GQA merge)
    int max_chunks = 0;
    size_t layer_elems = 0;   // elements of one layer of the K (or V) cache
    bool prev_decode = false; // the shard's last launch was a decode kernel (DecodeArgs::early)
    // baton_decode_step: the captured decode iteration, keyed by its I/O pointers
    // (a few I/O pointer sets, e.g. double-buffered staging; LRU replacement)
    static constexpr int kGraphs = 4;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t step_exec[kGraphs] = {nullptr, nullptr, nullptr, nullptr};
    const void *step_io[kGraphs][4] = {};
    unsigned long long step_used[kGraphs] = {0, 0, 0, 0};
    unsigned long long step_clock = 0;
    ~baton_state() {
        for (auto &e : step_exec)
            if (e) cudaGraphExecDestroy(e);
        if (cap_stream) cudaStreamDestroy(cap_stream);
    }
};

namespace {

thread_local int g_cuda_error = 0;

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return BATON_OK;
    g_cuda_error = (int)e;
    return BATON_E_CUDA;
}

bool shape_ok(const baton_shape *s) {
    if (!s) return false;
    return s->layers >= 1 && s->slots >= 1 && s->slots <= MAX_SLOTS && s->q_heads >= 1 &&
           s->kv_heads >= 1 && s->q_heads % s->kv_heads == 0 &&
           decode_supported_head_dim(s->head_dim) && s->max_ctx >= 16 && s->max_ctx % 16 == 0 &&
           s->max_ctx <= 65536;
}

size_t meta_bytes(const baton_shape *s) { return align256((1 + 2 * (size_t)s->slots) * 4); }
size_t ticket_region(const baton_shape *s) { return align256(decode_ticket_bytes(s->slots, s->q_heads)); }

cudaStream_t as_stream(void *s) { return static_cast<cudaStream_t>(s); }

__nv_bfloat16 *layer_ptr(void *base, const baton_state *st, int layer) {
    return static_cast<__nv_bfloat16 *>(base) + (size_t)layer * st->layer_elems;
}

// Transactional host mirror: a mutating call snapshots S/pad/lens/occ after its
// validation and restores them unless every launch of the call succeeded, so a
// failing call leaves the host mirror as it was (include/baton.h error contract).
struct MirrorTxn {
    baton_state *st;
    int S;
    std::vector<int32_t> pad, lens, occ;
    bool committed = false;
    explicit MirrorTxn(baton_state *s) : st(s), S(s->S), pad(s->pad), lens(s->lens), occ(s->occ) {}
    int commit(int r) {
        committed = r == BATON_OK;
        return r;
    }
    ~MirrorTxn() {
        if (committed) return;
        st->S = S;
        st->pad = pad;
        st->lens = lens;
        st->occ = occ;
    }
};

// Test-only fault injection (baton_debug_fail_launch): the n-th guarded splice
// launch from now is refused before it is enqueued, as a failed launch would be.
thread_local int g_fail_countdown = 0;
inline bool injected_failure() { return g_fail_countdown > 0 && --g_fail_countdown == 0; }
#define GUARDED(call) (injected_failure() ? cudaErrorLaunchFailure : (call))

int push_meta(baton_state *st, const std::vector<MaskOp> &ops, cudaStream_t s) {
    return cuda_status(GUARDED(launch_mask_splice(st->cfg.mask, st->sh.slots, st->sh.max_ctx, ops.data(),
                                          (int)ops.size(), st->d_S, st->d_lens, st->d_pad, st->S,
                                          st->lens.data(), st->pad.data(), s)));
}

}  // namespace

extern "C" {

size_t baton_decode_workspace_bytes(const baton_shape *s) {
    if (!shape_ok(s)) return 0;
    return ticket_region(s) + align256(decode_partial_bytes(s->slots, s->q_heads, s->head_dim, s->max_ctx));
}

size_t baton_workspace_bytes(const baton_shape *s) {
    if (!shape_ok(s)) return 0;
    // + a second partial buffer: consecutive layers of a decode step alternate them
    return meta_bytes(s) + baton_decode_workspace_bytes(s) +
           align256(decode_partial_bytes(s->slots, s->q_heads, s->head_dim, s->max_ctx));
}

int baton_create(const baton_config *cfg, void *stream, baton_state **out) {
    if (!cfg || !out || !shape_ok(&cfg->shape) || !cfg->k_cache || !cfg->v_cache || !cfg->mask ||
        !cfg->workspace)
        return BATON_E_INVALID;
    if (cfg->workspace_bytes < baton_workspace_bytes(&cfg->shape)) return BATON_E_INVALID;
    if ((reinterpret_cast<uintptr_t>(cfg->workspace) & 255) ||
        (reinterpret_cast<uintptr_t>(cfg->k_cache) & 15) ||
        (reinterpret_cast<uintptr_t>(cfg->v_cache) & 15) || (reinterpret_cast<uintptr_t>(cfg->mask) & 15))
        return BATON_E_INVALID;
    baton_state *st = new (std::nothrow) baton_state;
    if (!st) return BATON_E_INVALID;
    st->cfg = *cfg;
    st->sh = cfg->shape;
    const baton_shape &s = st->sh;
    st->pad.assign(s.slots, 0);
    st->lens.assign(s.slots, 0);
    st->occ.assign(s.slots, 0);
    uint8_t *ws = static_cast<uint8_t *>(cfg->workspace);
    st->d_S = reinterpret_cast<int32_t *>(ws);
    st->d_lens = st->d_S + 1;
    st->d_pad = st->d_lens + s.slots;
    // [meta | second partial buffer | tickets + counters | partial buffer]: the last
    // baton_decode_workspace_bytes are the stateless decode's layout (the binding hands
    // that tail to baton_decode_attention)
    const size_t p2 = align256(decode_partial_bytes(s.slots, s.q_heads, s.head_dim, s.max_ctx));
    st->partial2 = reinterpret_cast<float *>(ws + meta_bytes(&s));
    st->tickets = reinterpret_cast<int32_t *>(ws + meta_bytes(&s) + p2);
    st->partial = reinterpret_cast<float *>(ws + meta_bytes(&s) + p2 + ticket_region(&s));
    st->max_chunks = ceil_div(s.max_ctx, CHUNK);
    st->layer_elems = (size_t)s.slots * s.kv_heads * s.max_ctx * s.head_dim;
    cudaStream_t cs = as_stream(stream);
    cudaError_t e = cudaMemsetAsync(cfg->mask, 0, (size_t)s.slots * s.max_ctx, cs);
    if (e == cudaSuccess) e = cudaMemsetAsync(cfg->workspace, 0, baton_workspace_bytes(&s), cs);
    if (e != cudaSuccess) {
        delete st;
        return cuda_status(e);
    }
    *out = st;
    return BATON_OK;
}

void baton_destroy(baton_state *st) { delete st; }

int baton_device_meta(const baton_state *st, int32_t **S, int32_t **lens, int32_t **pad_start) {
    if (!st) return BATON_E_INVALID;
    if (S) *S = st->d_S;
    if (lens) *lens = st->d_lens;
    if (pad_start) *pad_start = st->d_pad;
    return BATON_OK;
}

int baton_query(const baton_state *st, int32_t *S, int32_t *pad_start, int32_t *lens,
                int32_t *occupied) {
    if (!st) return BATON_E_INVALID;
    const int B = st->sh.slots;
    if (S) *S = st->S;
    if (pad_start) std::memcpy(pad_start, st->pad.data(), B * 4);
    if (lens) std::memcpy(lens, st->lens.data(), B * 4);
    if (occupied) std::memcpy(occupied, st->occ.data(), B * 4);
    return BATON_OK;
}

// ---------------------------------------------------------------- a1
int baton_mask_update(baton_state *st, void *stream) {
    if (st) st->prev_decode = false;
    if (!st) return BATON_E_INVALID;
    if (st->S + 1 > st->sh.max_ctx) return BATON_E_CAPACITY;
    int r = cuda_status(launch_mask_update(st->cfg.mask, st->d_S, st->d_lens, st->sh.slots,
                                           st->sh.max_ctx, as_stream(stream)));
    if (r) return r;
    st->S += 1;
    for (int b = 0; b < st->sh.slots; ++b)
        if (st->occ[b]) st->lens[b] += 1;
    return BATON_OK;
}

// ---------------------------------------------------------------- a2
int baton_append_kv(baton_state *st, int layer, const void *k_new, const void *v_new, void *stream) {
    if (st) st->prev_decode = false;
    if (!st || !k_new || !v_new || layer < 0 || layer >= st->sh.layers) return BATON_E_INVALID;
    return cuda_status(launch_append_kv(layer_ptr(st->cfg.k_cache, st, layer),
                                        layer_ptr(st->cfg.v_cache, st, layer), k_new, v_new,
                                        st->d_lens, st->sh.slots, st->sh.kv_heads,
                                        st->sh.head_dim, st->sh.max_ctx, as_stream(stream)));
}

// ---------------------------------------------------------------- a3
int baton_decode_attention(const void *q, const void *k, const void *v, const uint8_t *mask,
                           const int32_t *lens, const int32_t *pad_start, void *out,
                           const baton_shape *shape, float scale, void *workspace,
                           size_t workspace_bytes, void *stream) {
    if (!q || !k || !v || !lens || !pad_start || !out || !workspace || !shape_ok(shape))
        return BATON_E_INVALID;
    if (workspace_bytes < baton_decode_workspace_bytes(shape)) return BATON_E_INVALID;
    if (!(scale > 0.f)) return BATON_E_INVALID;
    DecodeArgs a;
    a.q = q;
    a.k = k;
    a.v = v;
    a.mask = mask;
    a.lens = lens;
    a.pad = pad_start;
    a.out = out;
    a.tickets = static_cast<int32_t *>(workspace);
    a.counters = a.tickets + (size_t)shape->slots * shape->q_heads;
    a.partial = reinterpret_cast<float *>(static_cast<uint8_t *>(workspace) + ticket_region(shape));
    a.slots = shape->slots;
    a.q_heads = shape->q_heads;
    a.kv_heads = shape->kv_heads;
    a.head_dim = shape->head_dim;
    a.max_ctx = shape->max_ctx;
    a.max_chunks = ceil_div(shape->max_ctx, CHUNK);
    a.scale = scale;
    return cuda_status(launch_decode_attention(a, as_stream(stream)));
}

namespace {
// experiment builds: BATON_DEFER_MERGE=0 restores the in-layer merges for A/B runs
bool defer_merge_enabled() {
#if BATON_EXPERIMENTS
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_DEFER_MERGE");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
#else
    return true;
#endif
}

DecodeArgs layer_args(baton_state *st, int layer, const void *q, const void *k_new, const void *v_new,
                      void *out, bool early) {
    const baton_shape &s = st->sh;
    DecodeArgs a;
    a.q = q;
    a.k = layer_ptr(st->cfg.k_cache, st, layer);
    a.v = layer_ptr(st->cfg.v_cache, st, layer);
    a.k_new = k_new;
    a.v_new = v_new;
    a.mask = st->cfg.mask;
    a.lens = st->d_lens;
    a.pad = st->d_pad;
    a.out = out;
    a.tickets = st->tickets;
    a.counters = st->tickets + (size_t)s.slots * s.q_heads;
    a.partial = st->partial;
    a.slots = s.slots;
    a.q_heads = s.q_heads;
    a.kv_heads = s.kv_heads;
    a.head_dim = s.head_dim;
    a.max_ctx = s.max_ctx;
    a.max_chunks = st->max_chunks;
    a.scale = 1.0f / sqrtf((float)s.head_dim);
    a.early = early;
    return a;
}
}  // namespace

int baton_decode_layer(baton_state *st, int layer, const void *q, const void *k_new,
                       const void *v_new, void *out, void *stream) {
    if (!st || !q || !out || layer < 0 || layer >= st->sh.layers) return BATON_E_INVALID;
    if ((k_new == nullptr) != (v_new == nullptr)) return BATON_E_INVALID;
    // a2 fused into a3: one launch streams the cache and embeds the new token
    const int r = cuda_status(launch_decode_attention(
        layer_args(st, layer, q, k_new, v_new, out, st->prev_decode), as_stream(stream)));
    st->prev_decode = r == BATON_OK;
    return r;
}

int baton_decode_step(baton_state *st, const void *q, const void *k_new, const void *v_new,
                      void *out, void *stream) {
    if (st) st->prev_decode = false;
    if (!st || !q || !k_new || !v_new || !out) return BATON_E_INVALID;
    if (st->S + 1 > st->sh.max_ctx) return BATON_E_CAPACITY;
    const baton_shape &s = st->sh;
    const size_t qstride = (size_t)s.slots * s.q_heads * s.head_dim;
    const size_t kstride = (size_t)s.slots * s.kv_heads * s.head_dim;
    const void *io[4] = {q, k_new, v_new, out};
    int slot = -1;
    for (int i = 0; i < baton_state::kGraphs; ++i)
        if (st->step_exec[i] && std::memcmp(io, st->step_io[i], sizeof(io)) == 0) slot = i;
    if (slot < 0) {
        // capture: mask update + every layer's fused append/attention, chained with
        // programmatic dependent launch; the graph reads only device state
        slot = 0;
        for (int i = 1; i < baton_state::kGraphs; ++i)
            if (st->step_used[i] < st->step_used[slot]) slot = i;
        if (st->step_exec[slot]) {
            cudaGraphExecDestroy(st->step_exec[slot]);
            st->step_exec[slot] = nullptr;
        }
        cudaError_t e = cudaSuccess;
        if (!st->cap_stream) e = cudaStreamCreateWithFlags(&st->cap_stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_status(e);
        DecodeArgs probe = layer_args(st, 0, q, k_new, v_new, out, false);
        probe.dry = true;   // kernel attributes must be set outside the capture
        if ((e = launch_decode_attention(probe, st->cap_stream)) != cudaSuccess) return cuda_status(e);
        if ((e = cudaStreamBeginCapture(st->cap_stream, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
            return cuda_status(e);
        e = launch_mask_update(st->cfg.mask, st->d_S, st->d_lens, s.slots, s.max_ctx, st->cap_stream);
        // head_dim 128 (GQA and MHA): layer l's split-K merge runs at the start of
        // layer l+1's launch (buffers alternate by layer), so no merge sits in the
        // layer chain -- no combine kernel (GQA), no gpu-scope tickets on the
        // streaming warps (MHA); one combine after the last layer
        const bool defer = s.head_dim == 128 && defer_merge_enabled();
        DecodeArgs last{};
        for (int l = 0; l < s.layers && e == cudaSuccess; ++l) {
            const __nv_bfloat16 *ql = static_cast<const __nv_bfloat16 *>(q) + l * qstride;
            const __nv_bfloat16 *kl = static_cast<const __nv_bfloat16 *>(k_new) + l * kstride;
            const __nv_bfloat16 *vl = static_cast<const __nv_bfloat16 *>(v_new) + l * kstride;
            __nv_bfloat16 *ol = static_cast<__nv_bfloat16 *>(out) + l * qstride;
            // layer 0 follows the mask update (writes lens): no early prefetch
            DecodeArgs a = layer_args(st, l, ql, kl, vl, ol, l > 0);
            if (defer) {
                a.defer_merge = true;
                a.partial = (l & 1) ? st->partial2 : st->partial;
                if (l > 0) {
                    a.prev_partial = last.partial;
                    a.prev_out = last.out;
                }
            }
            e = launch_decode_attention(a, st->cap_stream);
            last = a;
        }
        if (defer && e == cudaSuccess && s.layers > 0) e = launch_gqa_combine(last, st->cap_stream);
        cudaGraph_t g = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(st->cap_stream, &g);
        if (e == cudaSuccess) e = e2;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&st->step_exec[slot], g, 0);
        if (g) cudaGraphDestroy(g);
        if (e != cudaSuccess) {
            st->step_exec[slot] = nullptr;
            return cuda_status(e);
        }
        std::memcpy(st->step_io[slot], io, sizeof(io));
    }
    st->step_used[slot] = ++st->step_clock;
    int r = cuda_status(cudaGraphLaunch(st->step_exec[slot], as_stream(stream)));
    if (r) return r;
    st->S += 1;   // host mirror of a1
    for (int b = 0; b < s.slots; ++b)
        if (st->occ[b]) st->lens[b] += 1;
    return BATON_OK;
}

// ---------------------------------------------------------------- NEXT-1
// The vector-SHAPING iteration (Baton without P&D): raw queries join
// with their whole prompt and every row's input is padded to width W.
int baton_shape_step(baton_state *st, int W, int n_new, const int32_t *new_slots, const int32_t *new_lens,
                     const void *q, const void *k_new, const void *v_new, void *out, void *stream) {
    if (st) st->prev_decode = false;
    if (!st || W < 1 || n_new < 0 || !q || !k_new || !v_new || !out) return BATON_E_INVALID;
    if (n_new > 0 && (!new_slots || !new_lens)) return BATON_E_INVALID;
    const baton_shape &s = st->sh;
    if (!prefill_supported(s.head_dim)) return BATON_E_INVALID;
    std::vector<int> newlen(s.slots, 0);
    for (int i = 0; i < n_new; ++i) {
        const int b = new_slots[i];
        if (b < 0 || b >= s.slots || newlen[b]) return BATON_E_INVALID;
        if (st->occ[b]) return BATON_E_SLOT_BUSY;
        if (new_lens[i] < 1 || new_lens[i] > W) return BATON_E_CAPACITY;
        newlen[b] = new_lens[i];
    }
    if (st->S + W > s.max_ctx) return BATON_E_CAPACITY;
    MirrorTxn txn(st);
    const int S0 = st->S;
    std::vector<MaskOp> ops;
    std::vector<int32_t> row0(s.slots, -1);
    for (int b = 0; b < s.slots; ++b) {
        if (st->occ[b]) {            // survivor: its token at column S0, then W-1 padding
            ops.push_back({MOP_SET_CELL, b, S0, 0});
            row0[b] = st->lens[b];
            st->lens[b] += W;
        } else if (newlen[b]) {      // new raw query: row := 0^S0 1^l 0^(W-l)
            ops.push_back({MOP_SET_ROW, b, S0, S0 + newlen[b]});
            row0[b] = 0;
            st->occ[b] = 1;
            st->pad[b] = S0;
            st->lens[b] = W;
        }
    }
    st->S = S0 + W;
    cudaStream_t cs = as_stream(stream);
    int r = push_meta(st, ops, cs);
    if (r) return r;
    // the W input tokens' K/V rows (reading C4: the cache grows by W as well)
    r = cuda_status(GUARDED(launch_shape_append(st->cfg.k_cache, st->cfg.v_cache, k_new, v_new, row0.data(), s.layers,
                                        s.slots, s.kv_heads, s.head_dim, s.max_ctx, W, cs)));
    if (r) return r;
    const size_t qstride = (size_t)s.slots * s.q_heads * W * s.head_dim;
    const float scale = 1.0f / sqrtf((float)s.head_dim);
    for (int l = 0; l < s.layers; ++l) {
        r = cuda_status(launch_extend_attention(
            static_cast<const __nv_bfloat16 *>(q) + l * qstride, layer_ptr(st->cfg.k_cache, st, l),
            layer_ptr(st->cfg.v_cache, st, l), static_cast<__nv_bfloat16 *>(out) + l * qstride, W, s.slots,
            s.q_heads, s.kv_heads, s.head_dim, s.max_ctx, st->d_lens, st->d_pad, st->cfg.mask, scale, cs));
        if (r) return r;
    }
    return txn.commit(BATON_OK);
}

// ---------------------------------------------------------------- a4
int baton_remove(baton_state *st, const int32_t *slots, int n, int32_t *released, void *stream) {
    if (st) st->prev_decode = false;
    if (!st || n < 0 || (n > 0 && !slots)) return BATON_E_INVALID;
    const int B = st->sh.slots;
    std::vector<char> seen(B, 0);
    for (int i = 0; i < n; ++i) {
        const int b = slots[i];
        if (b < 0 || b >= B || seen[b]) return BATON_E_INVALID;
        if (!st->occ[b]) return BATON_E_SLOT_EMPTY;
        seen[b] = 1;
    }
    MirrorTxn txn(st);
    std::vector<MaskOp> ops;
    for (int i = 0; i < n; ++i) {
        const int b = slots[i];
        ops.push_back({MOP_ZERO_ROW, b, 0, 0});
        st->occ[b] = 0;
        st->lens[b] = 0;
        st->pad[b] = 0;
    }
    // release [0 : min(index_i)] over occupied slots (everything if none, C5)
    int p = st->S;
    for (int b = 0; b < B; ++b)
        if (st->occ[b]) p = std::min(p, (int)st->pad[b]);
    if (p > 0) {
        ops.push_back({MOP_SHIFT_LEFT, -1, p, 0});
        for (int b = 0; b < B; ++b)
            if (st->occ[b]) st->pad[b] -= p;
        st->S -= p;
    }
    if (ops.empty()) {   // nothing removed, nothing to release
        if (released) *released = 0;
        return txn.commit(BATON_OK);
    }
    const int r = txn.commit(push_meta(st, ops, as_stream(stream)));
    if (released) *released = r == BATON_OK ? p : 0;
    return r;
}

// ---------------------------------------------------------------- a5
int baton_insert_many(baton_state *st, int n, const int32_t *slots, const void *const *k_pref,
                      const void *const *v_pref, const int32_t *lens, void *stream) {
    if (st) st->prev_decode = false;
    if (!st || n < 0) return BATON_E_INVALID;
    if (n == 0) return BATON_OK;
    if (!slots || !k_pref || !v_pref || !lens) return BATON_E_INVALID;
    const baton_shape &s = st->sh;
    std::vector<char> seen(s.slots, 0);
    for (int i = 0; i < n; ++i) {
        const int b = slots[i];
        if (b < 0 || b >= s.slots || seen[b] || !k_pref[i] || !v_pref[i]) return BATON_E_INVALID;
        if (st->occ[b]) return BATON_E_SLOT_BUSY;
        if (lens[i] < 1 || lens[i] > s.max_ctx) return BATON_E_CAPACITY;
        if ((reinterpret_cast<uintptr_t>(k_pref[i]) & 15) || (reinterpret_cast<uintptr_t>(v_pref[i]) & 15))
            return BATON_E_INVALID;
        seen[b] = 1;
    }
    MirrorTxn txn(st);
    std::vector<MaskOp> ops;
    std::vector<CopyJob> jobs;
    for (int i = 0; i < n; ++i) {
        const int b = slots[i];
        const int len = lens[i];
        if (len <= st->S) {   // P:L137 case 1: end-aligned
            st->pad[b] = st->S - len;
        } else {              // P:L137 case 2: expand on the left by e
            const int e = len - st->S;
            ops.push_back({MOP_SHIFT_RIGHT, -1, e, 0});
            for (int c = 0; c < s.slots; ++c)
                if (st->occ[c]) st->pad[c] += e;
            st->S = len;
            st->pad[b] = 0;
        }
        ops.push_back({MOP_SET_ROW, b, st->pad[b], st->S});
        st->occ[b] = 1;
        st->lens[b] = len;
        CopyJob j;
        j.src_k = k_pref[i];
        j.src_v = v_pref[i];
        j.dst_k = static_cast<__nv_bfloat16 *>(st->cfg.k_cache) + (size_t)b * s.kv_heads * s.max_ctx * s.head_dim;
        j.dst_v = static_cast<__nv_bfloat16 *>(st->cfg.v_cache) + (size_t)b * s.kv_heads * s.max_ctx * s.head_dim;
        j.src_hs = (int64_t)len * s.head_dim;
        j.src_ls = j.src_hs * s.kv_heads;
        j.dst_hs = (int64_t)s.max_ctx * s.head_dim;
        j.dst_ls = (int64_t)st->layer_elems;
        j.rows = len;
        j.pad_ = 0;
        jobs.push_back(j);
    }
    cudaStream_t cs = as_stream(stream);
    for (size_t i0 = 0; i0 < jobs.size(); i0 += MAX_SPLICE_JOBS) {
        const int nj = (int)std::min(jobs.size() - i0, (size_t)MAX_SPLICE_JOBS);
        int r = cuda_status(GUARDED(launch_kv_copy(jobs.data() + i0, nj, s.layers, s.kv_heads, s.head_dim, cs)));
        if (r) return r;
    }
    return txn.commit(push_meta(st, ops, cs));
}

int baton_insert(baton_state *st, int slot, const void *k_pref, const void *v_pref, int len,
                 void *stream) {
    const void *kp[1] = {k_pref};
    const void *vp[1] = {v_pref};
    const int32_t sl[1] = {slot};
    const int32_t ln[1] = {len};
    return baton_insert_many(st, 1, sl, kp, vp, ln, stream);
}

// ---------------------------------------------------------------- a6
int baton_extract(baton_state *st, int slot, void *k_out, void *v_out, void *stream) {
    if (st) st->prev_decode = false;
    if (!st || !k_out || !v_out) return BATON_E_INVALID;
    const baton_shape &s = st->sh;
    if (slot < 0 || slot >= s.slots) return BATON_E_INVALID;
    if (!st->occ[slot]) return BATON_E_SLOT_EMPTY;
    if ((reinterpret_cast<uintptr_t>(k_out) & 15) || (reinterpret_cast<uintptr_t>(v_out) & 15))
        return BATON_E_INVALID;
    const int len = st->lens[slot];
    CopyJob j;
    j.src_k = static_cast<__nv_bfloat16 *>(st->cfg.k_cache) + (size_t)slot * s.kv_heads * s.max_ctx * s.head_dim;
    j.src_v = static_cast<__nv_bfloat16 *>(st->cfg.v_cache) + (size_t)slot * s.kv_heads * s.max_ctx * s.head_dim;
    j.dst_k = k_out;
    j.dst_v = v_out;
    j.src_hs = (int64_t)s.max_ctx * s.head_dim;
    j.src_ls = (int64_t)st->layer_elems;
    j.dst_hs = (int64_t)len * s.head_dim;
    j.dst_ls = j.dst_hs * s.kv_heads;
    j.rows = len;
    j.pad_ = 0;
    return cuda_status(GUARDED(launch_kv_copy(&j, 1, s.layers, s.kv_heads, s.head_dim, as_stream(stream))));
}

// ---------------------------------------------------------------- a7
int baton_compact(baton_state *st, int n_active, int32_t *old_to_new, void *stream) {
    if (st) st->prev_decode = false;
    if (!st) return BATON_E_INVALID;
    const baton_shape &s = st->sh;
    if (n_active < 1 || n_active > s.slots) return BATON_E_INVALID;
    int n_occ_hi = 0, n_free_lo = 0;
    for (int b = 0; b < s.slots; ++b) {
        if (b >= n_active && st->occ[b]) ++n_occ_hi;
        if (b < n_active && !st->occ[b]) ++n_free_lo;
    }
    if (n_occ_hi > n_free_lo) return BATON_E_CAPACITY;
    MirrorTxn txn(st);
    std::vector<int32_t> src, dst;
    std::vector<CopyJob> jobs;
    std::vector<int32_t> o2n(s.slots);
    for (int b = 0; b < s.slots; ++b) o2n[b] = b;
    int f = 0;
    for (int b = n_active; b < s.slots; ++b) {
        if (!st->occ[b]) continue;
        while (st->occ[f]) ++f;   // lowest free slot < n_active (C19)
        src.push_back(b);
        dst.push_back(f);
        o2n[b] = f;
        CopyJob j;
        const size_t slot_elems = (size_t)s.kv_heads * s.max_ctx * s.head_dim;
        j.src_k = static_cast<__nv_bfloat16 *>(st->cfg.k_cache) + (size_t)b * slot_elems;
        j.src_v = static_cast<__nv_bfloat16 *>(st->cfg.v_cache) + (size_t)b * slot_elems;
        j.dst_k = static_cast<__nv_bfloat16 *>(st->cfg.k_cache) + (size_t)f * slot_elems;
        j.dst_v = static_cast<__nv_bfloat16 *>(st->cfg.v_cache) + (size_t)f * slot_elems;
        j.src_hs = j.dst_hs = (int64_t)s.max_ctx * s.head_dim;
        j.src_ls = j.dst_ls = (int64_t)st->layer_elems;
        j.rows = st->lens[b];
        j.pad_ = 0;
        jobs.push_back(j);
        st->occ[f] = 1;
        st->lens[f] = st->lens[b];
        st->pad[f] = st->pad[b];
        st->occ[b] = 0;
        st->lens[b] = 0;
        st->pad[b] = 0;
    }
    cudaStream_t cs = as_stream(stream);
    for (size_t i0 = 0; i0 < jobs.size(); i0 += MAX_SPLICE_JOBS) {
        const int nj = (int)std::min(jobs.size() - i0, (size_t)MAX_SPLICE_JOBS);
        int r = cuda_status(GUARDED(launch_kv_copy(jobs.data() + i0, nj, s.layers, s.kv_heads, s.head_dim, cs)));
        if (r) return r;
    }
    const int r = txn.commit(cuda_status(GUARDED(launch_mask_move(st->cfg.mask, s.slots, s.max_ctx, src.data(), dst.data(),
                                                                  (int)src.size(), st->d_S, st->d_lens, st->d_pad,
                                                                  st->S, st->lens.data(), st->pad.data(), cs))));
    // old_to_new is written only when the call succeeded (the mirror rolls back otherwise)
    if (r == BATON_OK && old_to_new) std::memcpy(old_to_new, o2n.data(), s.slots * 4);
    return r;
}

// ---------------------------------------------------------------- a8
int baton_prefill_attention(const void *q, const void *k, const void *v, void *out, int len,
                            const baton_shape *shape, float scale, void *stream) {
    if (!q || !k || !v || !out || !shape || len < 1 || !(scale > 0.f)) return BATON_E_INVALID;
    if (shape->q_heads < 1 || shape->kv_heads < 1 || shape->q_heads % shape->kv_heads ||
        !prefill_supported(shape->head_dim))
        return BATON_E_INVALID;
    for (const void *ptr : {q, k, v, (const void *)out})
        if (reinterpret_cast<uintptr_t>(ptr) & 15) return BATON_E_INVALID;
    return cuda_status(launch_prefill_attention(q, k, v, out, len, shape->q_heads, shape->kv_heads,
                                                shape->head_dim, scale, as_stream(stream)));
}

int baton_prefill_attention_varlen(const void *q, const void *k, const void *v, void *out,
                                   const int32_t *cu_lens, int n, const baton_shape *shape, float scale,
                                   void *stream) {
    if (!q || !k || !v || !out || !cu_lens || !shape || n < 1 || n > prefill_varlen_max_prompts() ||
        !(scale > 0.f))
        return BATON_E_INVALID;
    if (shape->q_heads < 1 || shape->kv_heads < 1 || shape->q_heads % shape->kv_heads ||
        !prefill_supported(shape->head_dim))
        return BATON_E_INVALID;
    if (cu_lens[0] != 0) return BATON_E_INVALID;
    int tiles = 0;
    for (int i = 0; i < n; ++i) {
        const int len = cu_lens[i + 1] - cu_lens[i];
        if (len < 1) return BATON_E_INVALID;
        tiles += (len + 127) / 128;
    }
    if (tiles > 1024) return BATON_E_INVALID;
    for (const void *ptr : {q, k, v, (const void *)out})
        if (reinterpret_cast<uintptr_t>(ptr) & 15) return BATON_E_INVALID;
    return cuda_status(launch_prefill_attention_varlen(q, k, v, out, cu_lens, n, shape->q_heads, shape->kv_heads,
                                                       shape->head_dim, scale, as_stream(stream)));
}

// ---------------------------------------------------------------- misc
const char *baton_error_string(int code) {
    switch (code) {
        case BATON_OK: return "ok";
        case BATON_E_INVALID: return "invalid argument";
        case BATON_E_SLOT_BUSY: return "slot busy";
        case BATON_E_SLOT_EMPTY: return "slot empty";
        case BATON_E_CAPACITY: return "capacity exceeded";
        case BATON_E_CUDA: return "CUDA error";
        default: return "unknown error";
    }
}

int baton_cuda_error(void) { return g_cuda_error; }

// Test-only (not in include/baton.h): refuse the n-th guarded splice launch
// (mask splice / mask move / K/V copy / shape append) of this thread from now on
// (n = 1: the next one; 0 disarms).  Used to check that a failing call leaves the
// host mirror and the device state unchanged.
int baton_debug_fail_launch(int n) {
    g_fail_countdown = n < 0 ? 0 : n;
    return BATON_OK;
}

// ---------------------------------------------------------------- harness keygen
int baton_keygen_tokens(void *out, const int32_t *qids, const int32_t *pos, int layers, int n_slots,
                        int heads, int head_dim, int kind, int layer0, uint64_t seed, int scale_exp,
                        void *stream) {
    if (!out || !qids || !pos || layers < 0 || n_slots < 0 || heads < 1 || heads > 64 ||
        head_dim < 1 || head_dim > 128 || kind < 0 || kind > 2 || layer0 < 0 || layer0 + layers > 128)
        return BATON_E_INVALID;
    return cuda_status(launch_keygen_tokens(out, qids, pos, layers, n_slots, heads, head_dim, kind,
                                            layer0, seed, scale_exp, as_stream(stream)));
}

int baton_keygen_history(void *out, int layers, int heads, int head_dim, int qid, int pos_begin,
                         int n, int kind, uint64_t seed, int scale_exp, int64_t head_stride,
                         int64_t layer_stride, void *stream) {
    if (!out || layers < 0 || layers > 128 || heads < 1 || heads > 64 || head_dim < 1 ||
        head_dim > 128 || qid < 0 || qid >= (1 << 20) || pos_begin < 0 || n < 0 ||
        pos_begin + n > 4096 || kind < 0 || kind > 2)
        return BATON_E_INVALID;
    return cuda_status(launch_keygen_history(out, layers, heads, head_dim, qid, pos_begin, n, kind,
                                             seed, scale_exp, head_stride, layer_stride,
                                             as_stream(stream)));
}

}  // extern "C"
