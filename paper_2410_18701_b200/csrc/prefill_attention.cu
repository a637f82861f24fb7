// prefill_attention.cu -- a8: causal attention of a newly inserted query over its
// own prompt, the "prefilling" that Baton decouples from decoding ("all
// original queries awaiting processing are initially prefilled by the model";
// P:L215 asynchronous P&D decoupling).  Row i of the output is the textbook
// SDPA of query token i over keys 0..i -- the decode attention of every
// prefix at once, a dense contraction, so it runs on the 5th-gen tensor cores.
//
// Work item = (q head, 128-query tile); a persistent grid of TWO CTAs per SM (~98 KB
// smem, 256 TMEM columns each) walks the items, so one CTA's softmax overlaps the
// other's MMAs and an item's Q load, first K/V tiles and first S MMAs run under the
// previous item's last P.V and epilogue.  Warp roles:
//   warp 4   TMA producer: per item the Q tile (128 x 128, SWIZZLE_128B; once the
//            previous item's last S MMA has read the buffer), then per 64-key tile K
//            and V, each through a 2-stage ring that runs on across items --
//            cp.async.bulk.tensor with mbarrier tx-counts
//   warp 5   MMA issuer (one elected thread): S(j) = Q K(j)^T (M=128, N=64, K=16 x8)
//            into TMEM buffer j&1, then O += P(j) V(j) (M=128, N=128, K=16 x4) with
//            P(j) read from TMEM (the "TS" form: P overwrites the first 32 columns of
//            its own S buffer, bf16 pairs), then S(j+2) into the buffer P(j) just
//            left -- the tensor pipe runs those in issue order, so S(j+2) cannot
//            overwrite P(j) before the P.V MMA has read it.  The softmax therefore
//            always finds the next scores ready.
//   warps 0-3 softmax: thread = query row; tcgen05.ld of its S row, causal mask,
//            online max/sum (exp2, lazy rescale), P -> bf16 -> tcgen05.st into TMEM,
//            O rescale in TMEM (tcgen05.ld/st) when the reference max moves, epilogue.
//
// The same kernel runs the EXTEND attention of a vector-shaping iteration
// (NEXT-1, launch_extend_attention): an item per (slot, q head, query
// tile); query row t of slot b is input token t of width W (q/out token-major,
// [slots][W][q_heads][D]: a 4-D Q map with a (64, 1, 128, 1) box), its keys are the
// slot's cache rows 0 .. off_b + t (off_b = lens_b - W, the rows before this
// iteration), and a key is also dropped where the paper's attention_mask is 0 (the
// mask bytes of each key tile ride in the V stage, which outlives the softmax of
// that tile).  Prefill is the case of one slot, off = 0 and no mask.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"
#include "tma.h"

namespace baton {
namespace {

constexpr int PF_M = 128;         // queries per tile (UMMA M, TMEM lanes)
constexpr int PF_N = 64;          // keys per tile (UMMA N of S, K of PV)
constexpr int PF_D = 128;         // head_dim
constexpr int PF_THREADS = 192;   // 4 softmax warps + producer warp + MMA warp
constexpr int VL_MAXP = 64;       // prompts per varlen prefill launch
constexpr int VL_MAXT = 1024;     // (prompt, query tile) entries per launch
constexpr int Q_BYTES = PF_M * PF_D * 2;        // 32 KB: two 16 KB swizzle regions (dims 0-63, 64-127)
constexpr int Q_REGION = Q_BYTES / 2;
constexpr int KV_BYTES = PF_N * PF_D * 2;       // 16 KB: two 8 KB regions
constexpr int KV_REGION = KV_BYTES / 2;

struct __align__(1024) PfSmem {
    uint8_t q[Q_BYTES];
    uint8_t k[2][KV_BYTES];
    uint8_t v[2][KV_BYTES];
    uint8_t mk[2][PF_N + 16];       // extend: mask bytes of the V stage's key tile
    uint64_t bar_q, q_empty, o_free, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_full[2], pv_done[2];
    uint32_t tmem_base;
};

using namespace tc;

// Debug counter (baton_debug_prefill_rescales): warps that took the lazy-rescale
// branch (O rows rescaled in TMEM).  One relaxed atomic per such warp-tile; the
// branch is rare by design (the reference max moves by > rescale_t log2 units).
__device__ unsigned long long g_pf_rescales = 0;

// Debug timeline (experiment builds; baton_debug_prefill_trace, scripts/trace_prefill.py):
// per CTA < PFT_CTAS, clock64 at [0] start, [1] end, and for the CTA's tiles t < 12:
// [2+5t] MMA issued S(t) (after its commits), [3+5t] softmax warp 0 holds S(t),
// [4+5t] softmax thread 0 published P(t), [5+5t] MMA thread's wait for P(t) returned,
// [6+5t] MMA issued P.V(t) (after its commits).
constexpr int PFT_CTAS = BATON_EXPERIMENTS ? 296 : 1, PFT_W = 62, PFT_T = 12;
__device__ int g_pft_on;
__device__ long long g_pft[PFT_CTAS][PFT_W];
#define PFT(t, f) \
    if (BATON_EXPERIMENTS && g_pft_on && blockIdx.x < PFT_CTAS && (t) < PFT_T) g_pft[blockIdx.x][2 + 5 * (t) + (f)] = clock64()

// packed fp32x2 FMA / add (SASS FFMA2 / FADD2): half the issue slots of the scalar ops
BATON_DEV float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t A, B, C, D;
    asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b.x), "f"(b.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(C) : "f"(c.x), "f"(c.y));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(C));
    float2 d;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(D));
    return d;
}
BATON_DEV float fmax3(float a, float b, float c) {   // SASS FMNMX3
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
BATON_DEV float2 fadd2(float2 a, float2 b) {
    uint64_t A, B, D;
    asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    float2 d;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(D));
    return d;
}

struct PfParams {
    int Hq, Hkv, len, n_mtiles;     // extend: len = W query rows per (slot, head)
    int n_items;                    // work items (prefill: entries x Hq; extend: n_mtiles x Hq x slots)
    float scale_log2;
    float rescale_t;                // lazy-rescale threshold (log2 units): P <= 2^rescale_t
    int skip;                       // prefill: skip causally dead 32-key chunks and dead warps (BATON_PF_SKIP)
    __nv_bfloat16 *out;
    // extend only (lens == nullptr for prefill)
    const int32_t *lens, *pad;      // device metadata AFTER the shaped mask update
    const uint8_t *mask;            // [slots][max_ctx]
    int max_ctx;
    // prefill only: prompts packed along the token axis (varlen), prompt i at rows
    // [vl_start[i], vl_start[i] + vl_len[i]); CTA c takes query tile vl_tile[c / Hq]
    // (prompt << 16 | m-tile, heaviest first) of q head c % Hq
    int32_t total;                  // packed token rows (the maps' second extent)
    int32_t vl_start[VL_MAXP], vl_len[VL_MAXP];
    uint32_t vl_tile[VL_MAXT];
};

// One work item = (prompt or slot, q head, 128-query tile).  Items are numbered
// heaviest first (prefill: the host's order; extend: slot-major, heavy tiles first
// within a (slot, head)).
struct PfItem {
    int b, h, mt, s0, len, off, kpad, n_kt;   // n_kt == 0: an empty extend slot (zero rows)
};

template <bool EXT>
BATON_DEV PfItem pf_item(const PfParams &p, int k) {
    PfItem it;
    if (EXT) {
        it.mt = p.n_mtiles - 1 - k % p.n_mtiles;
        it.h = (k / p.n_mtiles) % p.Hq;
        it.b = k / (p.n_mtiles * p.Hq);
        it.s0 = 0;
        it.len = p.len;
        const int lb = p.lens[it.b];
        if (lb <= 0) {
            it.off = it.kpad = it.n_kt = 0;
            return it;
        }
        it.off = lb - p.len;
        it.kpad = p.pad[it.b];
    } else {
        const uint32_t e = p.vl_tile[k / p.Hq];
        it.mt = (int)(e & 0xffff);
        it.h = k % p.Hq;
        it.b = 0;
        it.s0 = p.vl_start[e >> 16];
        it.len = p.vl_len[e >> 16];
        it.off = it.kpad = 0;
    }
    // key tiles up to the diagonal.  Varlen prefill: a tile may run past this prompt
    // into the next one's rows; those keys are past every query row of the tile
    // (causally masked, P = 0 exactly) and their V rows are finite
    it.n_kt = (it.off + min(it.mt * PF_M + PF_M, it.len) + PF_N - 1) / PF_N;
    return it;
}

// A persistent CTA's walk over its items: round r takes item r*G + c on even rounds
// and r*G + G-1-c on odd ones (a snake over the heaviest-first order, so the CTAs'
// loads even out), and positions (item, key tile j) in that order.  `seq` counts the
// non-empty items so far (the Q buffer's and the O accumulator's phases).
template <bool EXT>
struct PfWalk {
    const PfParams *p;
    int r, seq, j;
    bool valid;
    PfItem it;
    BATON_DEV int item_at(int rr) const {
        const int G = gridDim.x, c = blockIdx.x;
        return rr * G + ((rr & 1) ? G - 1 - c : c);
    }
    // first item at or after round rr (empty extend slots included: the softmax
    // warps write their zero rows)
    BATON_DEV void load(int rr) {
        r = rr;
        const int k = item_at(rr);
        valid = k < p->n_items;
        if (valid) it = pf_item<EXT>(*p, k);
        j = 0;
    }
    BATON_DEV void init(const PfParams *pp) {
        p = pp;
        seq = 0;
        load(0);
    }
    BATON_DEV void next_item() {
        if (it.n_kt > 0) ++seq;
        load(r + 1);
    }
    // next (item, tile) position, skipping empty items
    BATON_DEV void skip_empty() {
        while (valid && it.n_kt == 0) load(r + 1);
    }
    BATON_DEV void advance() {
        if (++j == it.n_kt) {
            next_item();
            skip_empty();
        }
    }
};

template <bool EXT>
__global__ void __launch_bounds__(PF_THREADS, 2)
prefill_attention_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ PfParams p) {
    extern __shared__ uint8_t smem_raw[];
    PfSmem &sm = *reinterpret_cast<PfSmem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr bool ext = EXT;

    if (BATON_EXPERIMENTS && g_pft_on && threadIdx.x == 0 && blockIdx.x < PFT_CTAS) g_pft[blockIdx.x][0] = clock64();
    if (threadIdx.x == 0) {
        mbar_init(&sm.bar_q, 1);
        mbar_init(&sm.q_empty, 1);
        mbar_init(&sm.o_free, 128);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.k_empty[s], 1);
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.v_empty[s], 1);
            mbar_init(&sm.s_full[s], 1);
            mbar_init(&sm.p_full[s], 128);
            mbar_init(&sm.pv_done[s], 1);
        }
        fence_mbar_init();
    }
    if (warp == 0) {   // TMEM: S/P buffers in columns [0,64) and [64,128), O in [128,256)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                         smem_u32(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t tS = tmem, tO = tmem + 128;

    if (warp == 4) {
        // ======================= TMA producer =======================
        // per item: the Q tile (once the previous item's last S MMA has read the Q
        // buffer), then its K and V tiles through the 2-stage rings; ring stages and
        // phases run on across items (t = this CTA's tile count)
        if (lane == 0) {
            prefetch_tmap(&tm_q);
            prefetch_tmap(&tm_k);
            prefetch_tmap(&tm_v);
            PfWalk<EXT> w;
            w.init(&p);
            w.skip_empty();
            int t = 0;
            for (; w.valid; w.next_item(), w.skip_empty()) {
                const PfItem &it = w.it;
                const int q0 = it.mt * PF_M;
                const int krow = it.b * p.Hkv + it.h * p.Hkv / p.Hq;
                if (w.seq > 0) mbar_wait(&sm.q_empty, (w.seq - 1) & 1);
                mbar_arrive_expect_tx(&sm.bar_q, Q_BYTES);
                if constexpr (EXT) {
                    tma_load_4d(sm.q, &tm_q, 0, it.h, q0, it.b, &sm.bar_q);
                    tma_load_4d(sm.q + Q_REGION, &tm_q, 64, it.h, q0, it.b, &sm.bar_q);
                } else {
                    tma_load_3d(sm.q, &tm_q, 0, it.s0 + q0, it.h, &sm.bar_q);
                    tma_load_3d(sm.q + Q_REGION, &tm_q, 64, it.s0 + q0, it.h, &sm.bar_q);
                }
                for (int j = 0; j < it.n_kt; ++j, ++t) {
                    const int s = t & 1;
                    if (t >= 2) mbar_wait(&sm.k_empty[s], ((t >> 1) + 1) & 1);   // S(t-2) done with K
                    mbar_arrive_expect_tx(&sm.k_full[s], KV_BYTES);
                    tma_load_3d(sm.k[s], &tm_k, 0, it.s0 + j * PF_N, krow, &sm.k_full[s]);
                    tma_load_3d(sm.k[s] + KV_REGION, &tm_k, 64, it.s0 + j * PF_N, krow, &sm.k_full[s]);
                    if (t >= 2) mbar_wait(&sm.v_empty[s], ((t >> 1) + 1) & 1);   // PV(t-2) done
                    uint32_t mbytes = 0;
                    size_t a0 = 0;
                    if (ext) {   // aligned superset of the tile's mask bytes (rows start 16-B aligned)
                        const size_t row0 = (size_t)it.b * p.max_ctx;
                        const size_t j0 = row0 + it.kpad + j * PF_N;
                        a0 = j0 & ~(size_t)15;
                        size_t need = (j0 + PF_N - a0 + 15) & ~(size_t)15;
                        if (a0 + need > row0 + p.max_ctx) need = row0 + p.max_ctx - a0;
                        mbytes = (uint32_t)need;
                    }
                    mbar_arrive_expect_tx(&sm.v_full[s], KV_BYTES + mbytes);
                    tma_load_3d(sm.v[s], &tm_v, 0, it.s0 + j * PF_N, krow, &sm.v_full[s]);
                    tma_load_3d(sm.v[s] + KV_REGION, &tm_v, 64, it.s0 + j * PF_N, krow, &sm.v_full[s]);
                    if (mbytes) bulk_g2s(sm.mk[s], p.mask + a0, mbytes, &sm.v_full[s]);
                }
            }
        }
    } else if (warp == 5) {
        // ======================= MMA issuer =======================
        // order over this CTA's whole tile stream: S(0), S(1), PV(0), S(2), PV(1), ...
        // S(t+2) goes into the TMEM buffer that P(t) occupies; it is issued after PV(t),
        // and the tensor pipe executes in issue order.  S(t+2) may be the next item's
        // first tile (its Q tile must have landed); an item's first PV overwrites O,
        // so it waits until the softmax warps have read the previous item's O out.
        // The whole warp walks the stream and waits; one elected lane issues (the
        // tcgen05 ops under elect.sync compile to single UTCHMMA/UTCBAR instructions,
        // not per-lane loops: the MMA thread's instruction stream paced the tile loop).
        {
            constexpr uint32_t idS = idesc_bf16(PF_M, PF_N, 0);   // B = K tile, K-major
            constexpr uint32_t idO = idesc_bf16(PF_M, PF_D, 1);   // A = P (TMEM, K-major), B = V tile, MN-major
            const uint32_t qa = smem_u32(sm.q);
            PfWalk<EXT> ws, wp;   // next S to issue, next PV to issue
            ws.init(&p);
            ws.skip_empty();
            wp.init(&p);
            wp.skip_empty();
            int ts = 0;
            auto issue_s = [&]() {
                const int b2 = ts & 1;
                if (ws.j == 0) {
                    mbar_wait(&sm.bar_q, ws.seq & 1);
                    tc_fence_after();
                }
                mbar_wait(&sm.k_full[b2], (ts >> 1) & 1);
                tc_fence_after();
                const uint32_t ka = smem_u32(sm.k[b2]);
                const bool last = ws.j == ws.it.n_kt - 1;
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {   // K = head_dim in steps of 16 (32 B)
                        umma_f16(tS + 64 * b2, smem_desc(qa + (k >> 2) * Q_REGION + (k & 3) * 32, 16, 1024),
                                 smem_desc(ka + (k >> 2) * KV_REGION + (k & 3) * 32, 16, 1024), idS, k > 0);
                    }
                    umma_commit(&sm.s_full[b2]);
                    PFT(ts, 0);
                    umma_commit(&sm.k_empty[b2]);
                    if (last) umma_commit(&sm.q_empty);   // the item's last S: Q may go
                }
                __syncwarp();
                ++ts;
                ws.advance();
            };
            if (ws.valid) issue_s();
            if (ws.valid) issue_s();
            for (int t = 0; wp.valid; ++t) {
                const int s = t & 1;
                mbar_wait(&sm.p_full[s], (t >> 1) & 1);           // P(t) in TMEM, O rescaled
                if (lane == 0) PFT(t, 3);
                mbar_wait(&sm.v_full[s], (t >> 1) & 1);
                if (wp.j == 0 && wp.seq > 0) mbar_wait(&sm.o_free, (wp.seq - 1) & 1);   // previous O read out
                tc_fence_after();
                const uint32_t va = smem_u32(sm.v[s]);
                const bool first = wp.j == 0;
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {   // K = 64 keys in steps of 16 (8 TMEM columns of bf16 pairs)
                        umma_f16_ts(tO, tS + 64 * s + 8 * k, smem_desc(va + k * 2048, KV_REGION, 1024), idO,
                                    (!first || k > 0));
                    }
                    umma_commit(&sm.pv_done[s]);
                    PFT(t, 4);
                    umma_commit(&sm.v_empty[s]);
                }
                __syncwarp();
                wp.advance();
                if (ws.valid) issue_s();
            }
        }
    } else {
        // ======================= softmax warps 0-3 =======================
        const int row = warp * 32 + lane;            // query row within the tile = TMEM lane
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        uint32_t pk[32];                              // P row (64 keys) packed bf16x2
        PfWalk<EXT> w;
        w.init(&p);
        int t = 0;                                    // this CTA's tile count (buffers, phases)
        for (; w.valid; w.next_item()) {
            const PfItem &it = w.it;
            const int q0 = it.mt * PF_M, qi = q0 + row, off = it.off;
            if (it.n_kt == 0) {   // extend, empty slot: zero output rows, nothing else
                for (int i = row; i < PF_M * PF_D / 8; i += 128) {
                    const int r = q0 + i / (PF_D / 8);
                    if (r < p.len)
                        reinterpret_cast<uint4 *>(p.out + (((size_t)it.b * p.len + r) * p.Hq + it.h) * PF_D)[i % (PF_D / 8)] =
                            make_uint4(0, 0, 0, 0);
                }
                continue;
            }
            float m = -INFINITY, l = 0.f;
            const int mrow = ext ? (int)(((size_t)it.b * p.max_ctx + it.kpad) & 15) : 0;   // mask byte offset
            // this warp's 32 rows are all past the prompt (prefill only: see the skips below)
            const bool rows_dead = !EXT && p.skip && q0 + warp * 32 >= it.len;
            for (int j = 0; j < it.n_kt; ++j, ++t) {
                const int sb = t & 1;
                const uint32_t tSj = tS + 64 * sb + lane_off;
                mbar_wait(&sm.s_full[sb], (t >> 1) & 1);
                if (threadIdx.x == 0) PFT(t, 1);
                // one thread observes PV(t-2)'s completion on its barrier: already done (S(t)
                // was issued after it and its commit covers every earlier MMA), so this never
                // blocks; it keeps every phase of pv_done waited on (compute-sanitizer
                // synccheck flags a phase completed with no wait; with all 128 threads
                // polling it cost ~1%)
                if (t >= 2 && threadIdx.x == 0) mbar_wait(&sm.pv_done[sb], ((t - 2) >> 1) & 1);
                tc_fence_after();
                const int kbase = j * PF_N;
                const bool diag = kbase + PF_N > off + q0;   // tile touches the causal diagonal
                const uint8_t *mk = sm.mk[sb] + mrow;
                if (ext) mbar_wait(&sm.v_full[sb], (t >> 1) & 1);   // this tile's mask bytes
                // Warp-uniform skips: a 32-key chunk whose first key is past this warp's
                // last row is causally dead for all 32 rows (the upper triangle of the
                // diagonal block); a warp whose rows are all past the prompt writes no
                // output.  Prefill only: in the extend kernel the extra branches made
                // ptxas spill.  Neither loads S, takes exponentials or touches m, l; a dead
                // chunk of a live warp gets P = 0 (its TMEM columns still hold S bits).
                const int wlast = off + q0 + warp * 32 + 31;
                const int live_c = rows_dead ? 0 : ((EXT || !p.skip) ? 2 : (kbase > wlast ? 0 : (kbase + 32 > wlast ? 1 : 2)));
                if (live_c > 0) {
                    uint32_t r[2][32];
                    tmem_ld32(tSj, r[0]);
                    tmem_ld32(tSj + 32, r[1]);
                    tmem_wait_ld();
                    // Masked keys become -inf in the RAW scores; the scale (> 0) is folded into
                    // the exponent (one FFMA + ex2 per key) and the row max is taken raw.  Tiles
                    // off the diagonal (and prefill has no mask) skip the per-key tests.
                    if (diag || ext) {
#pragma unroll
                        for (int c = 0; c < 2; ++c)
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                const bool dead = c >= live_c || (diag && kbase + c * 32 + i > off + qi) ||
                                                  (ext && mk[c * 32 + i] == 0);
                                if (dead) r[c][i] = __float_as_uint(-INFINITY);
                            }
                    }
                    float mx;
                    {   // row max: 3-input FMNMX3 in four independent chains
                        float a0 = -INFINITY, a1 = -INFINITY, a2 = -INFINITY, a3 = -INFINITY;
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            a0 = fmax3(a0, __uint_as_float(r[0][i]), __uint_as_float(r[0][i + 1]));
                            a1 = fmax3(a1, __uint_as_float(r[0][i + 2]), __uint_as_float(r[0][i + 3]));
                            a2 = fmax3(a2, __uint_as_float(r[1][i]), __uint_as_float(r[1][i + 1]));
                            a3 = fmax3(a3, __uint_as_float(r[1][i + 2]), __uint_as_float(r[1][i + 3]));
                        }
                        mx = fmax3(fmaxf(a0, a1), a2, a3);
                    }
                    mx *= p.scale_log2;   // -inf stays -inf
                    // Lazy rescale: P is taken relative to a reference max m that moves only
                    // when the row max exceeds it by more than rescale_t (log2 units), so P <=
                    // 2^rescale_t (exact in fp32 accumulation, same bf16 rounding of P) and the
                    // O rows in TMEM are rescaled only on those tiles, not whenever the max moves.
                    // A row may see only masked keys so far (extend: holes, padding): keep exp2
                    // finite -- ex2(-inf - 0) = 0.
                    const float m_new = (mx > m + p.rescale_t || m == -INFINITY) ? fmaxf(m, mx) : m;
                    const float mref = (m_new == -INFINITY) ? 0.f : m_new;
                    const float alpha = ex2(m - mref);
                    const float nref = -mref;
                    // the row sum adds the fp32 exponentials; the P.V MMA multiplies their bf16
                    // roundings (relative difference <= 2^-9 per key, far inside C13's 1e-2)
                    float2 rs2 = make_float2(0.f, 0.f);
                    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nr2 = make_float2(nref, nref);
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (c >= live_c) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) pk[c * 16 + i] = 0u;
                            continue;
                        }
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            float2 a = ffma2(make_float2(__uint_as_float(r[c][i]), __uint_as_float(r[c][i + 1])), sc2, nr2);
                            a.x = ex2(a.x);
                            a.y = ex2(a.y);
                            const __nv_bfloat162 b = __floats2bfloat162_rn(a.x, a.y);
                            rs2 = fadd2(rs2, a);
                            pk[c * 16 + i / 2] = *reinterpret_cast<const uint32_t *>(&b);
                        }
                    }
                    const float rs = rs2.x + rs2.y;
                    l = l * alpha + rs;
                    m = m_new;
                    // warp-uniform: tcgen05.ld/st are .sync.aligned (all 32 lanes converged)
                    if (j > 0 && __any_sync(FULL_MASK, alpha != 1.f)) {
                        // O is stable once PV(t-1) is done (PV(t-3) on that barrier completed
                        // before S(t-1), which this warp group already read: at most one phase behind)
                        mbar_wait(&sm.pv_done[(t - 1) & 1], ((t - 1) >> 1) & 1);
                        tc_fence_after();
                        if (lane == 0) atomicAdd(&g_pf_rescales, 1ull);
                        {
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                uint32_t o[32];
                                tmem_ld32(tO + lane_off + c * 32, o);
                                tmem_wait_ld();
#pragma unroll
                                for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                                tmem_st32(tO + lane_off + c * 32, o);
                            }
                            tmem_wait_st();
                        }
                    }
                } else if (!rows_dead) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) pk[i] = 0u;
                }
                // extend: cache rows past lens in this tile are stale memory (maybe NaN
                // bits); P is 0 there but 0 * NaN is not, so zero those V rows (whole 128-B
                // rows of both halves, swizzle-independent) before the P.V MMA reads them
                if (ext && kbase + PF_N > off + p.len) {
                    const int first = off + p.len - kbase;
                    for (int i = row; i < (PF_N - first) * 16; i += 128) {
                        const int rr = first + i / 16, ch = i % 16;
                        *reinterpret_cast<uint4 *>(sm.v[sb] + (ch >> 3) * KV_REGION + rr * 128 + (ch & 7) * 16) =
                            make_uint4(0, 0, 0, 0);
                    }
                    fence_async_smem();   // generic-proxy writes -> the tensor core's reads
                }
                // P row -> TMEM over the first 32 columns of this S buffer (bf16 pairs,
                // key 2c in the low half of column c): the A operand of PV(t).  Rows past
                // the prompt keep whatever the columns hold: their O rows are never written.
                if (!rows_dead) {
                    tmem_st32(tSj, pk);
                    tmem_wait_st();
                }
                tc_fence_before();
                mbar_arrive(&sm.p_full[sb]);
                if (threadIdx.x == 0) PFT(t, 2);
            }
            // epilogue: O / l -> bf16 once the item's last PV is done (the tensor pipe
            // completes in order); then O is released to the next item's first PV
            mbar_wait(&sm.pv_done[(t - 1) & 1], ((t - 1) >> 1) & 1);
            tc_fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            uint32_t o[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tO + lane_off + c * 32, o[c]);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&sm.o_free);
            if (qi < it.len) {
                __nv_bfloat16 *orow = EXT ? p.out + (((size_t)it.b * p.len + qi) * p.Hq + it.h) * PF_D
                                          : p.out + ((size_t)it.h * p.total + it.s0 + qi) * PF_D;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t wv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(o[c][2 * i]) * inv,
                                                                       __uint_as_float(o[c][2 * i + 1]) * inv);
                        wv[i] = *reinterpret_cast<const uint32_t *>(&b);
                    }
                    uint4 *o4 = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                    for (int i = 0; i < 4; ++i) o4[i] = make_uint4(wv[4 * i], wv[4 * i + 1], wv[4 * i + 2], wv[4 * i + 3]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (BATON_EXPERIMENTS && g_pft_on && threadIdx.x == 0 && blockIdx.x < PFT_CTAS) g_pft[blockIdx.x][1] = clock64();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

bool make_map(CUtensorMap *m, const void *base, int heads, int len, int box_rows) {
    const uint64_t dims[3] = {(uint64_t)PF_D, (uint64_t)len, (uint64_t)heads};
    const uint64_t strides[2] = {(uint64_t)PF_D * 2, (uint64_t)len * PF_D * 2};
    const uint32_t box[3] = {64, (uint32_t)box_rows, 1};
    return encode_bf16_map(m, base, 3, dims, strides, box);
}

}  // namespace

bool prefill_supported(int head_dim) { return head_dim == PF_D; }

namespace {
float g_rescale_override = -1.f;   // baton_debug_prefill_rescale_t
int g_grid_cap = 0;                // baton_debug_prefill_grid
// lazy-rescale threshold in log2 units: BATON_PF_RESCALE_T, default 8 (0 = rescale
// whenever the row max moves)
float pf_rescale_t() {
    if (g_rescale_override >= 0.f) return g_rescale_override;
    static float t = -1.f;
    if (t < 0.f) {
        const char *e = getenv("BATON_PF_RESCALE_T");
        t = e ? (float)atof(e) : 8.f;
        if (t < 0.f) t = 0.f;
    }
    return t;
}

// varlen item order (BATON_PF_ORDER): 0 = L2 panels (default), 1 = global heaviest
// first, 2 = prompt-major
int pf_order() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_PF_ORDER");
        v = e ? atoi(e) : 0;
        if (v < 0 || v > 2) v = 0;
    }
    return v;
}
int pf_panel_mb() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_PF_PANEL_MB");
        v = e ? atoi(e) : 64;
        if (v < 0) v = 0;
    }
    return v;
}

// warp-uniform skips of dead key chunks / rows in the prefill softmax (BATON_PF_SKIP=0: off)
int pf_skip() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_PF_SKIP");
        v = e ? (atoi(e) != 0) : 1;
    }
    return v;
}

bool pf_persist() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_PF_PERSIST");
        v = e ? atoi(e) != 0 : 1;
    }
    return v != 0;
}

cudaError_t launch_pf(const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv, const PfParams &p,
                      int slots, cudaStream_t s) {
    const size_t smem = sizeof(PfSmem) + 1024;
    PfParams pp = p;
    pp.rescale_t = pf_rescale_t();
    pp.skip = pf_skip();
    const bool ext = p.lens != nullptr;
    {
        cudaError_t e = ext ? ensure_smem_attr(prefill_attention_kernel<true>, smem)
                            : ensure_smem_attr(prefill_attention_kernel<false>, smem);
        if (e != cudaSuccess) return e;
    }
    // prefill: n_mtiles = number of (prompt, query tile) entries
    pp.n_items = p.n_mtiles * p.Hq * (ext ? slots : 1);
    // persistent grid: two CTAs per SM walk the items (BATON_PF_PERSIST=0: one CTA per
    // item, the round-1 launch shape, for A/B runs)
    int grid = pf_persist() ? std::min(pp.n_items, 2 * device_sms()) : pp.n_items;
    if (g_grid_cap > 0) grid = std::min(grid, g_grid_cap);   // tests: many items per CTA
    if (ext)
        prefill_attention_kernel<true><<<grid, PF_THREADS, smem, s>>>(mq, mk, mv, pp);
    else
        prefill_attention_kernel<false><<<grid, PF_THREADS, smem, s>>>(mq, mk, mv, pp);
    return cudaGetLastError();
}
}  // namespace

int prefill_varlen_max_prompts() { return VL_MAXP; }

namespace {
// The FA4-layout kernel (prefill_fa4.cu) is an experiment: measured slower than this
// file's kernel on every prompt shape, so the product prefill is
// this file's kernel; experiment builds select FA4 with BATON_PF_KERNEL=2
bool use_fa4() {
#if BATON_EXPERIMENTS
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_PF_KERNEL");
        v = e ? atoi(e) : 1;
    }
    return v == 2;
#else
    return false;
#endif
}
}  // namespace

// The varlen launch's work list: the (prompt, query tile) entries of n packed prompts,
// in the order the persistent grid walks them (x q heads, heads fastest).  Returns the
// number of entries, or -1 for an invalid cu_lens / too many entries.  Host only.
static int pf_plan(const int32_t *cu_lens, int n, int kv_heads, int head_dim, PfParams &p) {
    if (n < 1 || n > VL_MAXP || cu_lens[0] != 0) return -1;
    int ne = 0;
    for (int i = 0; i < n; ++i) {
        const int len = cu_lens[i + 1] - cu_lens[i];
        if (len < 1) return -1;
        p.vl_start[i] = cu_lens[i];
        p.vl_len[i] = len;
        const int nm = (len + PF_M - 1) / PF_M;
        if (ne + nm > VL_MAXT || nm > 0xffff) return -1;
        for (int mt = 0; mt < nm; ++mt) p.vl_tile[ne++] = ((uint32_t)i << 16) | (uint32_t)mt;
    }
    // cost of an entry: its key tiles up to the diagonal
    auto cost = [&](uint32_t e) {
        const int len = p.vl_len[e >> 16], q0 = (int)(e & 0xffff) * PF_M;
        return (std::min(q0 + PF_M, len) + PF_N - 1) / PF_N;
    };
    const int order_mode = pf_order();
    if (order_mode == 1) {   // global heaviest first (round 1)
        std::stable_sort(p.vl_tile, p.vl_tile + ne, [&](uint32_t a, uint32_t b) { return cost(a) > cost(b); });
    } else if (order_mode == 2) {   // prompt-major: longest prompt first, its tiles heaviest first
        std::stable_sort(p.vl_tile, p.vl_tile + ne, [&](uint32_t a, uint32_t b) {
            const int la = p.vl_len[a >> 16], lb = p.vl_len[b >> 16];
            if (la != lb) return la > lb;
            if ((a >> 16) != (b >> 16)) return (a >> 16) < (b >> 16);
            return (a & 0xffff) > (b & 0xffff);
        });
    } else {
        // L2 panels (default): prompts longest first are cut into panels of <= 64 MB of
        // K/V (BATON_PF_PANEL_MB; 0 = one panel) of the 126 MB L2; entries run panel by
        // panel, heaviest first within a panel.  The items in flight then share a
        // panel's prompts, so each (prompt, kv head)'s K/V is read from HBM about once
        // and reused from L2 by its other query tiles, while within a panel the
        // heaviest-first order keeps the CTAs' loads even.  A batch that fits one panel
        // keeps the round-1 order.
        int order[VL_MAXP], panel[VL_MAXP];
        for (int i = 0; i < n; ++i) order[i] = i;
        std::stable_sort(order, order + n, [&](int a, int b) { return p.vl_len[a] > p.vl_len[b]; });
        const double cap = (double)pf_panel_mb() * (1 << 20);
        double acc = 0.0;
        int pid = 0;
        for (int i = 0; i < n; ++i) {
            const double kv = 4.0 * p.vl_len[order[i]] * kv_heads * head_dim;   // K + V bytes
            if (cap > 0 && acc > 0 && acc + kv > cap) {
                ++pid;
                acc = 0.0;
            }
            acc += kv;
            panel[order[i]] = pid;
        }
        std::stable_sort(p.vl_tile, p.vl_tile + ne, [&](uint32_t a, uint32_t b) {
            const int pa = panel[a >> 16], pb = panel[b >> 16];
            if (pa != pb) return pa < pb;
            return cost(a) > cost(b);
        });
    }
    return ne;
}

cudaError_t launch_prefill_attention_varlen(const void *q, const void *k, const void *v, void *out,
                                            const int32_t *cu_lens, int n, int q_heads, int kv_heads,
                                            int head_dim, float scale, cudaStream_t s) {
    if (head_dim != PF_D || n < 1 || n > VL_MAXP || cu_lens[0] != 0) return cudaErrorInvalidValue;
#if BATON_EXPERIMENTS
    if (use_fa4()) return launch_prefill_fa4_varlen(q, k, v, out, cu_lens, n, q_heads, kv_heads, scale, pf_rescale_t(), s);
#endif
    PfParams p{};
    const int ne = pf_plan(cu_lens, n, kv_heads, head_dim, p);
    if (ne < 0) return cudaErrorInvalidValue;
    const int total = cu_lens[n];
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, q, q_heads, total, PF_M) || !make_map(&mk, k, kv_heads, total, PF_N) ||
        !make_map(&mv, v, kv_heads, total, PF_N))
        return cudaErrorInvalidValue;
    p.Hq = q_heads;
    p.Hkv = kv_heads;
    p.len = 0;
    p.total = total;
    p.n_mtiles = ne;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.out = static_cast<__nv_bfloat16 *>(out);
    p.lens = nullptr;
    return launch_pf(mq, mk, mv, p, 1, s);
}

cudaError_t launch_prefill_attention(const void *q, const void *k, const void *v, void *out, int len,
                                     int q_heads, int kv_heads, int head_dim, float scale,
                                     cudaStream_t s) {
    if (len < 1) return cudaErrorInvalidValue;
    const int32_t cu[2] = {0, len};
    return launch_prefill_attention_varlen(q, k, v, out, cu, 1, q_heads, kv_heads, head_dim, scale, s);
}

cudaError_t launch_extend_attention(const void *q, const void *k_layer, const void *v_layer, void *out,
                                    int W, int slots, int q_heads, int kv_heads, int head_dim, int max_ctx,
                                    const int32_t *lens, const int32_t *pad, const uint8_t *mask,
                                    float scale, cudaStream_t s) {
    if (head_dim != PF_D || W < 1) return cudaErrorInvalidValue;
    CUtensorMap mq, mk, mv;
    // q: [slots][W][q_heads][D] (token-major) -> dims (D, q_heads, W, slots), box (64, 1, 128, 1)
    const uint64_t qd[4] = {(uint64_t)PF_D, (uint64_t)q_heads, (uint64_t)W, (uint64_t)slots};
    const uint64_t qs[3] = {(uint64_t)PF_D * 2, (uint64_t)q_heads * PF_D * 2, (uint64_t)W * q_heads * PF_D * 2};
    const uint32_t qb[4] = {64, 1, (uint32_t)PF_M, 1};
    // cache layer: [slots*kv_heads][max_ctx][D]
    if (!encode_bf16_map(&mq, q, 4, qd, qs, qb) || !make_map(&mk, k_layer, slots * kv_heads, max_ctx, PF_N) ||
        !make_map(&mv, v_layer, slots * kv_heads, max_ctx, PF_N))
        return cudaErrorInvalidValue;
    PfParams p{};
    p.Hq = q_heads;
    p.Hkv = kv_heads;
    p.len = W;
    p.n_mtiles = (W + PF_M - 1) / PF_M;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.out = static_cast<__nv_bfloat16 *>(out);
    p.lens = lens;
    p.pad = pad;
    p.mask = mask;
    p.max_ctx = max_ctx;
    return launch_pf(mq, mk, mv, p, slots, s);
}

}  // namespace baton

// Debug only (not part of include/baton.h).  baton_debug_prefill_rescales: the
// number of warp-tiles that rescaled O since the last reset (reset != 0 zeroes it;
// synchronous).  baton_debug_prefill_rescale_t: override the lazy-rescale
// threshold (log2 units; < 0 restores BATON_PF_RESCALE_T / the default 8).
extern "C" long long baton_debug_prefill_rescales(int reset) {
    unsigned long long v = 0;
    if (cudaMemcpyFromSymbol(&v, baton::g_pf_rescales, sizeof(v)) != cudaSuccess) return -1;
    if (reset) {
        const unsigned long long z = 0;
        if (cudaMemcpyToSymbol(baton::g_pf_rescales, &z, sizeof(z)) != cudaSuccess) return -1;
    }
#if BATON_EXPERIMENTS
    const long long f = baton::fa4_rescale_count(reset != 0);
    return f < 0 ? -1 : (long long)v + f;
#else
    return (long long)v;
#endif
}
extern "C" int baton_debug_prefill_rescale_t(float t) {
    baton::g_rescale_override = t;
    return 0;
}
// baton_debug_prefill_grid: cap the persistent grid at g CTAs (g <= 0 restores the
// default), so tests can make every CTA walk many items (results are independent of
// which CTA runs an item).
extern "C" int baton_debug_prefill_grid(int g) {
    baton::g_grid_cap = g > 0 ? g : 0;
    return 0;
}
// baton_debug_prefill_plan: the varlen launch's (prompt, query tile) work list in walk
// order, each entry prompt << 16 | tile, for n packed prompts (cu_lens[n + 1], host);
// writes at most cap entries to `out` and returns their total count, or -1 if the
// launch would refuse cu_lens.  Host only (no device work): CPU tests check the order.
extern "C" int baton_debug_prefill_plan(const int32_t *cu_lens, int n, int kv_heads, int head_dim, uint32_t *out,
                                        int cap) {
    static baton::PfParams p;   // ~9 KB: not on the caller's stack
    const int ne = baton::pf_plan(cu_lens, n, kv_heads, head_dim, p);
    for (int i = 0; i < ne && i < cap; ++i) out[i] = p.vl_tile[i];
    return ne;
}
// baton_debug_prefill_trace (experiment builds): on >= 0 switches the per-tile clock64
// timeline on (zeroed) or off; host != nullptr copies it out ([CTA][62] int64).
extern "C" int baton_debug_prefill_trace(int on, void *host, size_t bytes) {
#if !BATON_EXPERIMENTS
    (void)on;
    (void)host;
    (void)bytes;
    return -1;
#else
    if (host && cudaMemcpyFromSymbol(host, baton::g_pft, bytes < sizeof(baton::g_pft) ? bytes : sizeof(baton::g_pft)) !=
                    cudaSuccess)
        return -1;
    if (on >= 0) {
        if (on) {
            static long long zero[baton::PFT_CTAS][baton::PFT_W];
            cudaMemcpyToSymbol(baton::g_pft, zero, sizeof(zero));
        }
        if (cudaMemcpyToSymbol(baton::g_pft_on, &on, sizeof(int)) != cudaSuccess) return -1;
    }
    return 0;
#endif
}
