// decode_attention.cu -- a3 of the hot path: masked decode attention over the
// slot-relative KV cache (§2.1 SDPA; P:L52/P:L132 decode with the latest
// single token; masked padding skipped).
//
// Design:
//   * work item = (slot b, q head h, chunk c) of BATON_CHUNK = 256 keys counted
//     from the slot's live start (fixed chunking -> batch-invariant results);
//     items ordered (b, c, h), distributed round-robin over persistent CTAs
//     (2 per SM).
//   * one PRODUCER warp (one elected lane) streams 64-key K and V tiles plus the
//     tile's mask bytes and, on an item's first tile, the query vector into a
//     3-stage shared-memory ring with 1-D bulk copies (cp.async.bulk -> UBLKCP,
//     the TMA engine), completion tracked by mbarrier transaction counts.
//     Rows outside [0, lens) are never requested.
//   * four CONSUMER warps each own 16 rows of a tile.  A warp reads two 256-B
//     rows per 16-B-per-lane shared load (conflict-free), forms partial dot
//     products on 8 dims per lane and finishes them with a transposing
//     butterfly (8 shuffles per 16 keys), keeps an online softmax (running max
//     m, running sum l, unnormalised o) in fp32, exp2-based with scale*log2(e)
//     folded into q.
//   * an item's four warp states are merged in shared memory; a single-chunk
//     query writes its bf16 output directly, otherwise the chunk partial
//     (m, l, o[D]) goes to the workspace and the LAST CTA to finish a
//     (b, h) (atomic ticket) merges the chunk partials in ascending chunk order.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "gqa_merge.cuh"
#include "sched.cuh"

namespace baton {

// Debug timeline (off unless baton_debug_mha_trace(1, ...) was called); launch l
// writes slot l % MT_L.  Per CTA: [0] enter [1] work list built [2] consumer exit
// [3] items [4] smid [5] producer past the wait; per item k < 6: [8+4k] w, [9+4k]
// first copy issued, [10+4k] first tile ready, [11+4k] epilogue done.
constexpr int MT_L = BATON_EXPERIMENTS ? 8 : 1, MT_CTAS = BATON_EXPERIMENTS ? 1024 : 1, MT_W = 32;
__device__ int g_mtrace_on;
__device__ long long g_mtrace[MT_L][MT_CTAS][MT_W];
static int g_mtrace_launch = 0;
BATON_DEV long long mtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

namespace {

constexpr int ROWS_PER_WARP = 16;
// (consumer warps, ring stages, CTAs per SM) are template parameters; the default
// for head_dim 128 is (2, 2, 5): 32-key tiles, many small independent CTAs -- the
// sweep showed resident-CTA parallelism beats deeper rings (see launch table).

constexpr int F_FIRST = 1, F_LAST = 2, F_END = 4, F_WRITE = 8;

__device__ __forceinline__ int ceil_div_dev(int L) { return (L + CHUNK - 1) / CHUNK; }

struct StageDesc {
    int32_t b, h, c, nrows, flags, moff, nchunks, wrow;
};

template <int D, int TILE>
struct __align__(16) Stage {
    __nv_bfloat16 k[TILE * D];
    __nv_bfloat16 v[TILE * D];
    __nv_bfloat16 q[D < 8 ? 8 : D];
    uint8_t mask[TILE + 16];
    StageDesc desc;
};

struct Params {
    const __nv_bfloat16 *q, *k, *v;
    const __nv_bfloat16 *k_new, *v_new;      // fused append (nullable)
    __nv_bfloat16 *k_w, *v_w;                // cache base for the append write-back
    int32_t *counters;                       // dynamic work counter (workspace)
    const uint8_t *mask;
    const int32_t *lens, *pad;
    __nv_bfloat16 *out;
    float *partial;
    int32_t *tickets;
    int B, Hq, Hkv, max_ctx, max_chunks;
    float scale_log2;
    bool early;                              // prefetch before griddepcontrol.wait
    bool defer;                              // decode step: leave split-K merges to the next launch
    const float *prev_partial;               // ... and merge the previous layer's (head_dim 128)
    __nv_bfloat16 *prev_out;
    int trace_slot;                          // debug timeline slot
};

template <int D, int CWARPS, int STAGES>
struct Smem {
    Stage<D, CWARPS * ROWS_PER_WARP> st[STAGES];
    uint64_t full[STAGES], empty[STAGES];
    WorkSched ws;
    float red_o[2][CWARPS][D];
    float red_m[2][CWARPS], red_l[2][CWARPS];
    uint64_t part_bar;
};

template <int D, int CWARPS, int STAGES, int MINB>
__global__ void __launch_bounds__((CWARPS + 1) * 32, MINB) decode_attention_kernel(const Params p) {
    constexpr int TILE = CWARPS * ROWS_PER_WARP;
    constexpr int THREADS = (CWARPS + 1) * 32;
    constexpr int LPR = D / 8;                 // lanes per key row (16 B of bf16 per lane)
    constexpr int RPL = 32 / LPR;              // rows per warp-wide load
    constexpr int NL = ROWS_PER_WARP / RPL;    // loads per lane per tile
    static_assert(NL * 2 == LPR || (LPR == 2 && NL == 1), "row mapping");

    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem<D, CWARPS, STAGES> &sm = *reinterpret_cast<Smem<D, CWARPS, STAGES> *>(smem_raw);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const bool trace = BATON_EXPERIMENTS && g_mtrace_on && blockIdx.x < MT_CTAS;
    long long *tr = g_mtrace[p.trace_slot][trace ? blockIdx.x : 0];
    if (trace && threadIdx.x == 0) {
        tr[0] = mtimer();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        tr[4] = smid;
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], CWARPS);
        }
        mbar_init(&sm.part_bar, CWARPS * 32);
        fence_mbar_init();
    }
    __syncthreads();
    // PDL.  Without p.early everything below reads lens/pad/mask/cache only after
    // the previous kernel completed.  With p.early (the host saw that the previous
    // launch was a decode kernel, which writes none of lens/pad/mask and no cache
    // row but lens-1) the producer builds the work list and streams the first ring
    // of K/V tiles of a statically assigned first item BEFORE the wait, overlapping
    // the previous layer's tail; q, the appended row and every write wait for it.
    // Every thread waits before it triggers, so when any kernel starts, all
    // launches two or more back in the stream have completed.
    if (!p.early) {
        griddep_wait();
        griddep_launch_dependents();
    }

    if (warp == CWARPS) {
        // ============================ producer warp ============================
        sched_build(sm.ws, p.lens, p.pad, p.B, p.Hq, lane);
        // The whole warp walks the work list (identical state in every lane; the dynamic
        // counter is drawn by lane 0 and broadcast) and waits on the ring; one elected
        // lane per tile writes the stage descriptor and issues its copies, so the bulk
        // copies compile to single UBLKCP instructions rather than per-lane loops.
        if (trace && lane == 0) tr[1] = mtimer();
        int titem = 0;
        const int total = sched_total(sm.ws, p.Hq);
        const uint64_t pol = policy_evict_first();
        int stage = 0;
        uint32_t phase = 0;
        int b = 0;
        bool waited = !p.early;
        const __nv_bfloat16 *late_q = nullptr;   // q of a tile issued before the wait
        int late_stage = 0, issued = 0;
        auto flush = [&]() {
            griddep_wait();
            griddep_launch_dependents();
            waited = true;
            if (trace && lane == 0) tr[5] = mtimer();
            if (late_q && elect_one()) bulk_g2s(sm.st[late_stage].q, late_q, D * 2, &sm.full[late_stage]);
            __syncwarp();
            late_q = nullptr;
        };
        auto draw = [&]() {   // next dynamic item, one atomic per warp
            int v = 0;
            if (lane == 0) v = sched_next(p.counters);
            return (int)gridDim.x + __shfl_sync(FULL_MASK, v, 0);
        };
        // items [0, gridDim.x) are static (CTA i takes item i: no counter before the
        // wait), the rest are handed out by the dynamic counter
        int w = blockIdx.x;
        int w_next = waited ? draw() : -1;
        while (w < total) {
            int c, h;
            sched_item(sm.ws, w, p.Hq, b, c, h);
            const int L = sm.ws.lens[b];
            const int nch = ceil_div_dev(L);
            const int g = h * p.Hkv / p.Hq;
            const int r0 = c * CHUNK;
            const int rows = min(CHUNK, L - r0);
            const size_t head_off = ((size_t)(b * p.Hkv + g) * p.max_ctx + r0) * D;
            const __nv_bfloat16 *kb = p.k + head_off;
            const __nv_bfloat16 *vb = p.v + head_off;
            const int ntiles = (rows + TILE - 1) / TILE;
            // fused append (a2): the item holding row L-1 takes the new token's k/v
            // from k_new/v_new; the first q head of the kv group writes it to the cache
            const bool app = p.k_new != nullptr && c == nch - 1;
            if (trace && titem < 6 && lane == 0) {
                tr[8 + 4 * titem] = w;
                tr[9 + 4 * titem] = mtimer();
            }
            ++titem;
            for (int t = 0; t < ntiles; ++t) {
                const int nr = min(TILE, rows - t * TILE);
                const bool app_tile = app && t == ntiles - 1;
                // row L-1 may still be written by the previous (same-layer) kernel
                if (!waited && (issued == STAGES || r0 + t * TILE + nr == L)) flush();
                mbar_wait(&sm.empty[stage], phase ^ 1);
                Stage<D, TILE> &st = sm.st[stage];
                uint32_t bytes = 2u * nr * D * 2;
                int moff = 0;
                uint32_t mbytes = 0;
                const uint8_t *msrc = nullptr;
                if (p.mask) {
                    // aligned superset of the tile's mask bytes (row start is 16-B aligned)
                    const size_t row0 = (size_t)b * p.max_ctx;
                    const size_t j0 = row0 + sm.ws.pad[b] + r0 + t * TILE;
                    const size_t a0 = j0 & ~(size_t)15;
                    const size_t row_end = row0 + p.max_ctx;
                    size_t need = (j0 + nr - a0 + 15) & ~(size_t)15;
                    if (a0 + need > row_end) need = row_end - a0;
                    msrc = p.mask + a0;
                    mbytes = (uint32_t)need;
                    moff = (int)(j0 - a0);
                    bytes += mbytes;
                }
                if (t == 0) bytes += D * 2;
                const __nv_bfloat16 *qsrc = p.q + (size_t)(b * p.Hq + h) * D;
                if (elect_one()) {
                    st.desc.b = b;
                    st.desc.h = h;
                    st.desc.c = c;
                    st.desc.nrows = nr;
                    st.desc.flags = (t == 0 ? F_FIRST : 0) | (t == ntiles - 1 ? F_LAST : 0) |
                                    (app_tile && h * p.Hkv % p.Hq == 0 ? F_WRITE : 0);
                    st.desc.moff = moff;
                    st.desc.nchunks = nch;
                    st.desc.wrow = L - 1;
                    mbar_arrive_expect_tx(&sm.full[stage], bytes);
                    const int ncache = app_tile ? nr - 1 : nr;
                    if (ncache > 0) {
                        bulk_g2s_evict_first(st.k, kb + (size_t)t * TILE * D, ncache * D * 2, &sm.full[stage], pol);
                        bulk_g2s_evict_first(st.v, vb + (size_t)t * TILE * D, ncache * D * 2, &sm.full[stage], pol);
                    }
                    if (app_tile) {   // (always after the wait: see the flush above)
                        const size_t nb = ((size_t)b * p.Hkv + g) * D;
                        bulk_g2s(st.k + (nr - 1) * D, p.k_new + nb, D * 2, &sm.full[stage]);
                        bulk_g2s(st.v + (nr - 1) * D, p.v_new + nb, D * 2, &sm.full[stage]);
                    }
                    if (mbytes) bulk_g2s(st.mask, msrc, mbytes, &sm.full[stage]);
                    if (t == 0 && waited) bulk_g2s(st.q, qsrc, D * 2, &sm.full[stage]);
                }
                __syncwarp();
                if (t == 0 && !waited) {
                    late_q = qsrc;
                    late_stage = stage;
                }
                ++issued;
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (!waited) flush();
            if (w_next < 0) w_next = draw();
            w = w_next;
            w_next = w < total ? draw() : total;
        }
        if (!waited) flush();
        if (lane == 0) sched_done(p.counters);
        mbar_wait(&sm.empty[stage], phase ^ 1);
        if (lane != 0) return;
        sm.st[stage].desc.flags = F_END;
        mbar_arrive(&sm.full[stage]);
        return;
    }

    // ============================ consumer warps ============================
    if (p.early) {
        griddep_wait();
        griddep_launch_dependents();
    }
    // decode step (head_dim 128): the previous layer's split-K merge, its partials
    // complete and visible now; the producer keeps filling the ring meanwhile
    if constexpr (D == 128) {
        if (p.prev_partial)
            gqa_merge_pairs(p.lens, p.prev_partial, p.prev_out, p.B, p.Hq, p.max_chunks,
                            blockIdx.x * CWARPS + warp, gridDim.x * CWARPS, lane);
    }
    // Empty slots produce a zero output row (C6).
    for (int b = blockIdx.x; b < p.B; b += gridDim.x) {
        if (p.lens[b] <= 0) {
            uint4 *o = reinterpret_cast<uint4 *>(p.out + (size_t)b * p.Hq * D);
            for (int i = threadIdx.x; i < p.Hq * D / 8; i += CWARPS * 32) o[i] = make_uint4(0, 0, 0, 0);
        }
    }
    const int g = lane / LPR;        // row group within a warp-wide load
    const int s = lane % LPR;        // 16-B column chunk: dims [8s, 8s+8)
    const int my_row = (s >> 1) * RPL + g;   // row whose score this lane ends up holding
    float qf[8], o[8];
    float m = -INFINITY, l = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = qf[i] = 0.f;

    int stage = 0;
    uint32_t phase = 0;
    int rb = 0;                  // merge buffer of the current item
    uint32_t part_phase = 0;     // parity of part_bar (tracked by warp 0)
    int citem = 0;
    while (true) {
        mbar_wait(&sm.full[stage], phase);
        Stage<D, TILE> &st = sm.st[stage];
        const StageDesc d = st.desc;
        if (d.flags & F_END) break;
        if (trace && threadIdx.x == 0 && (d.flags & F_FIRST) && citem < 6) tr[10 + 4 * citem] = mtimer();
        if (d.flags & F_FIRST) {
            const uint4 qv = *reinterpret_cast<const uint4 *>(st.q + s * 8);
            const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                qf[2 * i] = bf16lo(qw[i]) * p.scale_log2;
                qf[2 * i + 1] = bf16hi(qw[i]) * p.scale_log2;
            }
            m = -INFINITY;
            l = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = 0.f;
        }
        const int base = warp * ROWS_PER_WARP;
        if ((d.flags & F_WRITE) && warp == (d.nrows - 1) / ROWS_PER_WARP && lane < D / 8) {
            // a2: the new token's k/v (already staged in smem) into cache row lens-1
            const size_t dst = (((size_t)d.b * p.Hkv + d.h * p.Hkv / p.Hq) * p.max_ctx + d.wrow) * D;
            reinterpret_cast<uint4 *>(p.k_w + dst)[lane] =
                reinterpret_cast<const uint4 *>(st.k + (d.nrows - 1) * D)[lane];
            reinterpret_cast<uint4 *>(p.v_w + dst)[lane] =
                reinterpret_cast<const uint4 *>(st.v + (d.nrows - 1) * D)[lane];
        }
        if (base < d.nrows) {
            // ---- scores: partial dots over this lane's 8 dims, NL rows
            float part[NL];
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const uint4 kv =
                    *reinterpret_cast<const uint4 *>(st.k + (base + i * RPL + g) * D + s * 8);
                const uint32_t kw[4] = {kv.x, kv.y, kv.z, kv.w};
                float acc = 0.f;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc = fmaf(qf[2 * j], bf16lo(kw[j]), acc);
                    acc = fmaf(qf[2 * j + 1], bf16hi(kw[j]), acc);
                }
                part[i] = acc;
            }
            // ---- transposing butterfly: after it, lane holds the full dot of my_row
#pragma unroll
            for (int step = 0, n = NL, msk = LPR / 2; n > 1; ++step, n >>= 1, msk >>= 1) {
                const bool upper = (lane & msk) != 0;
#pragma unroll
                for (int k2 = 0; k2 < n / 2; ++k2) {
                    const float send = upper ? part[k2] : part[k2 + n / 2];
                    const float keep = upper ? part[k2 + n / 2] : part[k2];
                    part[k2] = keep + __shfl_xor_sync(FULL_MASK, send, msk);
                }
            }
            float sc = part[0] + __shfl_xor_sync(FULL_MASK, part[0], 1);
            const int row = base + my_row;
            bool valid = row < d.nrows;
            if (p.mask) valid = valid && (st.mask[d.moff + (valid ? row : 0)] != 0);
            sc = valid ? sc : -INFINITY;
            float tmax = sc;
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(FULL_MASK, tmax, o2));
            const float m_new = fmaxf(m, tmax);
            if (m_new != -INFINITY) {
                const float alpha = ex2(m - m_new);     // m = -inf -> 0
                const float pe = ex2(sc - m_new);       // masked -> 0
                l = l * alpha + pe;
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] *= alpha;
                const bool all_valid = __all_sync(FULL_MASK, valid);
#pragma unroll
                for (int i = 0; i < NL; ++i) {
                    const int src = g * LPR + 2 * i;
                    float pi = __shfl_sync(FULL_MASK, pe, src);
                    uint4 vv = *reinterpret_cast<const uint4 *>(st.v + (base + i * RPL + g) * D + s * 8);
                    if (!all_valid) {
                        const bool vi = __shfl_sync(FULL_MASK, valid, src);
                        if (!vi) {
                            pi = 0.f;
                            vv = make_uint4(0, 0, 0, 0);
                        }
                    }
                    const uint32_t vw[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        o[2 * j] = fmaf(pi, bf16lo(vw[j]), o[2 * j]);
                        o[2 * j + 1] = fmaf(pi, bf16hi(vw[j]), o[2 * j + 1]);
                    }
                }
                m = m_new;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[stage]);
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }

        if (d.flags & F_LAST) {
            // ---- merge the four warp states of this item (double-buffered smem:
            // a warp can start the next item while others still read this one)
            float lsum = l;
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) lsum += __shfl_xor_sync(FULL_MASK, lsum, o2);
            lsum *= 0.5f;   // every row's weight is held by two lanes
#pragma unroll
            for (int mk = LPR; mk < 32; mk <<= 1)
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] += __shfl_xor_sync(FULL_MASK, o[i], mk);
            if (lane < LPR) {
#pragma unroll
                for (int i = 0; i < 8; ++i) sm.red_o[rb][warp][s * 8 + i] = o[i];
            }
            if (lane == 0) {
                sm.red_m[rb][warp] = m;
                sm.red_l[rb][warp] = lsum;
            }
            named_bar_sync(1, CWARPS * 32);
            const int t = threadIdx.x;
            float M = -INFINITY;
#pragma unroll
            for (int w2 = 0; w2 < CWARPS; ++w2) M = fmaxf(M, sm.red_m[rb][w2]);
            const size_t bh = (size_t)d.b * p.Hq + d.h;
            for (int dd = t; dd < D; dd += CWARPS * 32) {
                float Lt = 0.f, Ot = 0.f;
#pragma unroll
                for (int w2 = 0; w2 < CWARPS; ++w2) {
                    const float mw = sm.red_m[rb][w2];
                    const float f = (mw == -INFINITY) ? 0.f : ex2(mw - M);
                    Lt = fmaf(f, sm.red_l[rb][w2], Lt);
                    Ot = fmaf(f, sm.red_o[rb][w2][dd], Ot);
                }
                if (d.nchunks == 1) {
                    p.out[bh * D + dd] = __float2bfloat16_rn(Lt > 0.f ? Ot / Lt : 0.f);
                } else {
                    float *pp = p.partial + (bh * p.max_chunks + d.c) * (D + PREC_PAD);
                    pp[dd] = Ot;
                    if (dd == 0) {
                        pp[D] = M;
                        pp[D + 1] = Lt;
                    }
                }
            }
            rb ^= 1;
            if (d.nchunks > 1 && !p.defer) {
                // publish the partial: every thread arrives (release, non-blocking);
                // warp 0 alone waits, then one gpu-scope acq_rel ticket.  The CTA that
                // draws the last ticket merges the chunks in ascending chunk order.
                // (Making the last chunk's item the merger instead was measured: it
                // waits for sibling chunks still streaming -- profiles/r01_mha_trace.md.)
                mbar_arrive(&sm.part_bar);
                if (warp == 0) {
                    mbar_wait(&sm.part_bar, part_phase);
                    part_phase ^= 1;
                    int last = 0;
                    if (lane == 0) last = atom_add_acq_rel_gpu(&p.tickets[bh], 1) == d.nchunks - 1;
                    __syncwarp();
                    last = __shfl_sync(FULL_MASK, last, 0);
                    if (last) {
                        // two passes (global max, weighted sums); loads 8 chunks deep so
                        // the merge costs two L2 round trips for up to 8 chunks
                        const float *pc = p.partial + bh * p.max_chunks * (D + PREC_PAD);
                        const int nch = d.nchunks;
                        float Mc = -INFINITY;
                        for (int c0 = 0; c0 < nch; c0 += 8) {
                            float mv[8];
#pragma unroll
                            for (int j2 = 0; j2 < 8; ++j2)
                                mv[j2] = c0 + j2 < nch ? __ldcg(pc + (c0 + j2) * (D + PREC_PAD) + D) : -INFINITY;
#pragma unroll
                            for (int j2 = 0; j2 < 8; ++j2) Mc = fmaxf(Mc, mv[j2]);
                        }
                        constexpr int NJ = (D + 31) / 32;
                        float Lc = 0.f, Oc[NJ];
#pragma unroll
                        for (int j = 0; j < NJ; ++j) Oc[j] = 0.f;
                        for (int c0 = 0; c0 < nch; c0 += 8) {
                            float fv[8], lv[8], ov[8][NJ];
#pragma unroll
                            for (int j2 = 0; j2 < 8; ++j2) {
                                const bool ok = c0 + j2 < nch;
                                const float *r = pc + (ok ? c0 + j2 : 0) * (D + PREC_PAD);
                                fv[j2] = ok ? __ldcg(r + D) : -INFINITY;
                                lv[j2] = ok ? __ldcg(r + D + 1) : 0.f;
#pragma unroll
                                for (int j = 0; j < NJ; ++j)
                                    ov[j2][j] = (ok && j * 32 + lane < D) ? __ldcg(r + j * 32 + lane) : 0.f;
                            }
#pragma unroll
                            for (int j2 = 0; j2 < 8; ++j2) {
                                const float f = (fv[j2] == -INFINITY) ? 0.f : ex2(fv[j2] - Mc);
                                Lc = fmaf(f, lv[j2], Lc);
#pragma unroll
                                for (int j = 0; j < NJ; ++j) Oc[j] = fmaf(f, ov[j2][j], Oc[j]);
                            }
                        }
                        const float inv = Lc > 0.f ? 1.f / Lc : 0.f;
#pragma unroll
                        for (int j = 0; j < NJ; ++j)
                            if (j * 32 + lane < D) p.out[bh * D + j * 32 + lane] = __float2bfloat16_rn(Oc[j] * inv);
                        if (lane == 0) p.tickets[bh] = 0;
                    }
                }
            }
            if (trace && threadIdx.x == 0 && citem < 6) tr[11 + 4 * citem] = mtimer();
            ++citem;
        }
    }
    if (trace && threadIdx.x == 0) {
        tr[2] = mtimer();
        tr[3] = citem;
    }
}

template <int D, int CW, int ST, int MINB>
cudaError_t launch_d(const DecodeArgs &a, cudaStream_t s) {
    const int num_sms = device_sms();
    const size_t smem = sizeof(Smem<D, CW, ST>);
    {
        cudaError_t e = ensure_smem_attr(decode_attention_kernel<D, CW, ST, MINB>, smem);
        if (e != cudaSuccess) return e;
    }
    if (a.dry) return cudaSuccess;
    Params p;
    p.q = static_cast<const __nv_bfloat16 *>(a.q);
    p.k = static_cast<const __nv_bfloat16 *>(a.k);
    p.v = static_cast<const __nv_bfloat16 *>(a.v);
    p.k_new = static_cast<const __nv_bfloat16 *>(a.k_new);
    p.v_new = static_cast<const __nv_bfloat16 *>(a.v_new);
    p.k_w = static_cast<__nv_bfloat16 *>(const_cast<void *>(a.k));
    p.v_w = static_cast<__nv_bfloat16 *>(const_cast<void *>(a.v));
    p.counters = a.counters;
    p.mask = a.mask;
    p.lens = a.lens;
    p.pad = a.pad;
    p.out = static_cast<__nv_bfloat16 *>(a.out);
    p.partial = a.partial;
    p.tickets = a.tickets;
    p.B = a.slots;
    p.Hq = a.q_heads;
    p.Hkv = a.kv_heads;
    p.max_ctx = a.max_ctx;
    p.max_chunks = a.max_chunks;
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.early = a.early;
    p.defer = a.defer_merge && D == 128;
    p.prev_partial = D == 128 ? a.prev_partial : nullptr;
    p.prev_out = static_cast<__nv_bfloat16 *>(a.prev_out);
    p.trace_slot = g_mtrace_launch++ % MT_L;
    return launch_pdl(decode_attention_kernel<D, CW, ST, MINB>, dim3(MINB * num_sms),
                      dim3((CW + 1) * 32), smem, s, p);
}

// head_dim 128 pipeline variants (consumer warps, ring stages, CTAs per SM), chosen
// by BATON_MHA_VARIANT for sweeps in experiment builds; 0 is the default.
int mha_variant() {
#if BATON_EXPERIMENTS
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_MHA_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
#else
    return 0;
#endif
}

}  // namespace

size_t decode_partial_bytes(int slots, int q_heads, int head_dim, int max_ctx) {
    return (size_t)slots * q_heads * ceil_div(max_ctx, CHUNK) * (head_dim + PREC_PAD) * sizeof(float);
}
size_t decode_ticket_bytes(int slots, int q_heads) {
    return (size_t)slots * q_heads * sizeof(int32_t) + 2 * sizeof(int32_t);   // + work counters
}
bool decode_supported_head_dim(int d) { return d == 16 || d == 32 || d == 64 || d == 128; }

cudaError_t launch_decode_attention(const DecodeArgs &a, cudaStream_t s) {
    if (gqa_supported(a.q_heads, a.kv_heads, a.head_dim)) return launch_decode_gqa(a, s);
    switch (a.head_dim) {
        case 16: return launch_d<16, 4, 3, 2>(a, s);
        case 32: return launch_d<32, 4, 3, 2>(a, s);
        case 64: return launch_d<64, 4, 3, 2>(a, s);
        case 128:
            switch (mha_variant()) {
                // measured on the cfg2 t0 state (profiles/r01_mha_sweep.md), us/launch:
                // (4,3,2) 66.2  (4,6,1) 93.6  (8,3,1) 82.3  (4,2,3) 59.8  (2,3,3) 64.2
                // (2,2,5) 58.7  (2,2,4) 59.2  (1,4,5) 64.6  (3,2,3) 60.8
                // late round 1, on the current kernel: (4,2,3) beats (2,2,5) by 2% on
                // configs[1] and by 24% on the stress shard (few items per CTA), ties on
                // 13B churn -> the default (profiles/r01_mha_sweep.md)
#if BATON_EXPERIMENTS
                case 1: return launch_d<128, 4, 3, 2>(a, s);
                case 5: return launch_d<128, 2, 2, 5>(a, s);
                case 6: return launch_d<128, 2, 2, 4>(a, s);
#endif
                default: return launch_d<128, 4, 2, 3>(a, s);
            }
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace baton

// Debug only (not part of include/baton.h): MHA decode timeline on/off + copy out
// ([MT_L][MT_CTAS][MT_W] int64, see g_mtrace).
extern "C" int baton_debug_mha_trace(int on, void *host, size_t bytes) {
#if !BATON_EXPERIMENTS
    (void)on;
    (void)host;
    (void)bytes;
    return -1;   // timelines exist in experiment builds only
#endif
    if (host) {
        if (cudaMemcpyFromSymbol(host, baton::g_mtrace, bytes < sizeof(baton::g_mtrace) ? bytes : sizeof(baton::g_mtrace)) != cudaSuccess)
            return -1;
    }
    if (on >= 0) {
        if (on) {
            static long long zero[baton::MT_L][baton::MT_CTAS][baton::MT_W];
            cudaMemcpyToSymbol(baton::g_mtrace, zero, sizeof(zero));
        }
        if (cudaMemcpyToSymbol(baton::g_mtrace_on, &on, sizeof(int)) != cudaSuccess) return -1;
    }
    return 0;
}
