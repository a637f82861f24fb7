// decode_gqa_tc.cu -- a3 for GQA groups of 8 on the 5th-gen tensor cores
// (tcgen05.mma, TMEM accumulators), BATON_GQA_VARIANT=20.
//
// Why: the mma.sync kernel (decode_gqa.cu) is bound by its consumer warps, not by
// HBM.  Its per-tile phase clocks (profiles/r01_gqa_engine_sweep.md) show ~600 of
// ~1250 cycles spent feeding K through ldmatrix and the MMA chain.  Here the tensor
// core reads K, V and q straight from shared memory, and the warps only run the
// softmax.
//
//   work item = (slot b, kv head g, 256-key chunk c) -- the same list, dynamic
//   schedule, early prefetch and split-K partial layout as decode_gqa.cu; tile =
//   128 keys (2 tiles per full chunk).
//   S^T[128 keys x 16]  = K[128 x 128 dims] . Q^T[128 x 16 (8 real heads)]
//                         UMMA M=128, N=16, A = K (K-major), B = q (K-major)
//   O^T[128 dims x 16] += V^T[128 dims x 128 keys] . P^T[128 keys x 16]
//                         UMMA M=128, N=16, A = V (MN-major), B = P^T (K-major)
//   TWO softmax warpgroups (warps 0-3, 4-7) take alternate ITEMS, so two tiles'
//   softmax chains run at once (each group: its own S double buffer, P buffer,
//   O accumulator in TMEM, barriers and smem exchange).  Thread = key (S) / dim
//   (O) lane.  Per tile: tcgen05.ld of the key's 8 head scores, per-head tile max
//   by redux.sync on order-preserving ints + a 4-warp exchange, online softmax
//   (exp2), P^T -> bf16 in the SW128 K-major layout, O rescale in TMEM only when a
//   head's max moved.  Row sums are kept per thread and reduced once per item.
//   warp 8: TMA producer (K/V 2-D boxes 64 dims x 128 rows, q 64 x 16, mask bytes,
//   the appended row).  Three MMA issuer warps with blocking waits (each a converged
//   warp issuing its tcgen05 ops from one elect.sync lane): warp 9
//   issues S for the tiles in order (into the owning group's free S buffer) and
//   hands each group its tiles through small smem queues; warps 10 and 11 issue
//   P.V for group 0 and group 1 as soon as that group published P, so one group's
//   slow tile never holds up the other's MMAs.  Warp 9 also patches the appended
//   row into the swizzled K/V tile before the S MMA (and writes it to the cache).
#include <cstdlib>

#include "common.cuh"
#include "gqa_merge.cuh"
#include "kernels.h"
#include "sched.cuh"
#include "tcgen05.cuh"
#include "tma.h"

namespace baton {

// Debug timeline (off unless baton_debug_gqa_tc_trace(1, ...)): per CTA [0] enter,
// [1] exit; per tile j < 16: [4+4j] MMA issued S(j), [5+4j] softmax holds S(j),
// [6+4j] softmax published P(j), [7+4j] MMA issued P.V(j).
constexpr int TT_CTAS = BATON_EXPERIMENTS ? 160 : 1, TT_W = 68;
__device__ int g_tt_on;
__device__ long long g_tt[2][TT_CTAS][TT_W];

namespace {
using namespace tc;
BATON_DEV long long tt_now() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int D = 128, GS = 8, NH = 16;      // UMMA N = 16 heads (8 real)
constexpr int TK = 128;                      // keys per tile
constexpr int TAIL = 32;                     // rows per TMA box of a short (last) tile
constexpr int STAGES = 3;
constexpr int KREG = TK * 128;               // 16 KB: a 64-dim half of a K or V tile
constexpr int QREG = NH * 128;               // 2 KB: a 64-dim half of the q tile
constexpr int PREG = NH * 128;               // 2 KB: 64 keys of P^T
constexpr int THREADS = 384;                 // 2 softmax warpgroups, producer, 3 MMA issuers
constexpr int F_FIRST = 1, F_LAST = 2, F_END = 4, F_WRITE = 8;

struct TDesc {
    int32_t b, g, c, nrows, flags, moff, nchunks, wrow, item, stage;
};

struct __align__(1024) TStage {
    uint8_t k[2 * KREG];
    uint8_t v[2 * KREG];
    uint8_t mask[TK + 16];
    __nv_bfloat16 knew[D], vnew[D];
    TDesc desc;
};

struct PvEntry {
    int32_t stage, flags;
    int32_t bh0, multi;                      // publish: (slot, kv group) ticket of a split item's last tile
};

struct __align__(1024) TSmem {
    TStage st[STAGES];
    uint8_t q[2][2 * QREG];                  // per group (= item parity)
    uint8_t p[2][2 * PREG];                  // P^T per group
    uint64_t full[STAGES], empty[STAGES], q_empty[2];
    uint64_t s_full[2][2], s_free[2][2], p_full[2], o_done[2];   // [group][S buffer] / [group]
    uint64_t pub[2];                         // publish: the group's partials are written
    TDesc gq[2][2];                          // the group's tile queue, per S buffer
    PvEntry pvq[2][4];                       // the P.V issuer's queue, per group
    WorkSched ws;
    int32_t red[2][2][4][GS];                // [group][tile parity][warp][head] tile max (encoded)
    float lsum[2][4][GS];
    int32_t last[2];
    float mf[2][32][GS], ml[2][32][GS];      // fused merge: chunk m / l per head (<= 32 chunks)
    uint32_t tmem_base;
};

struct TParams {
    const __nv_bfloat16 *q;
    const __nv_bfloat16 *k_new, *v_new;
    __nv_bfloat16 *k_w, *v_w;
    int32_t *counters;
    const uint8_t *mask;
    const int32_t *lens, *pad;
    __nv_bfloat16 *out;
    float *partial;
    int32_t *tickets;
    int B, Hq, Hkv, max_ctx, max_chunks;
    float scale_log2;
    bool early;
    bool fused;                              // in-kernel split-K merge (no combine launch)
    const float *prev_partial;               // decode step: merge the previous layer's split-K
    __nv_bfloat16 *prev_out;                 // partials at the start (DecodeArgs::defer_merge)
    bool publish;                            // count published chunks per (slot, kv group) for a
                                             // combine that merges as soon as a group is complete
};

BATON_DEV void tma_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// float <-> int with the same ordering (for redux.sync.max)
BATON_DEV int f2o(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
BATON_DEV float o2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }
// byte offset of 16-B chunk c (0..15) of row r in a SW128 K-major tile of `reg` bytes per half
BATON_DEV uint32_t swz(int r, int c, int reg) {
    return (uint32_t)((c >> 3) * reg + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// <= 144 registers: 384 x 144 = 55K leaves room on the SM for a combine CTA (128 x 72),
// so the next layer's CTA can enter while this layer drains (PDL early phase)
__global__ void __maxnreg__(144)
decode_gqa_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                     const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap32,
                     const __grid_constant__ CUtensorMap vmap32, const TParams p) {
    extern __shared__ uint8_t smem_raw[];
    TSmem &sm = *reinterpret_cast<TSmem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool trace = BATON_EXPERIMENTS && g_tt_on && blockIdx.x < TT_CTAS;
    long long *tr = g_tt[(p.prev_partial && p.partial > p.prev_partial) ? 1 : 0][trace ? blockIdx.x : 0];
    if (trace && threadIdx.x == 0) tr[0] = tt_now();

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&sm.q_empty[g], 1);
            mbar_init(&sm.p_full[g], 128);
            mbar_init(&sm.o_done[g], 1);
            mbar_init(&sm.pub[g], 128);
            for (int b2 = 0; b2 < 2; ++b2) {
                mbar_init(&sm.s_full[g][b2], 2);      // S MMAs done + queue entry written
                mbar_init(&sm.s_free[g][b2], 128);
            }
        }
        fence_mbar_init();
    }
    if (warp == 0) {   // TMEM: S[g][b] at 32g + 16b, O[g] at 64 + 16g
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                         smem_u32(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // P^T rows 8..15 (heads that do not exist) stay zero
    for (int i = threadIdx.x; i < 4 * PREG / 16; i += THREADS) reinterpret_cast<uint4 *>(sm.p)[i] = make_uint4(0, 0, 0, 0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    if (!p.early) {
        griddep_wait();
        griddep_launch_dependents();
    }

    if (warp == 8) {
        // ============================ producer ============================
        sched_build(sm.ws, p.lens, p.pad, p.B, p.Hkv, lane);
        // The whole warp walks the work list (identical state in every lane; the dynamic
        // counter is drawn by lane 0 and broadcast) and waits on the ring; one elected
        // lane per tile writes the stage descriptor and issues its loads, so the TMA ops
        // compile to single UTMALDG instructions rather than per-lane loops.
        {
            if (elect_one()) {
                prefetch_tmap(&kmap);
                prefetch_tmap(&vmap);
                prefetch_tmap(&qmap);
                prefetch_tmap(&kmap32);
                prefetch_tmap(&vmap32);
            }
            __syncwarp();
            const int total = sched_total(sm.ws, p.Hkv);
            int stage = 0, b = 0, item = 0, issued = 0;
            uint32_t phase = 0;
            bool waited = !p.early;
            int late_row = -1, late_stage = 0, late_par = 0;
            auto load_q = [&](int row, int s, int par) {
                tma_2d(sm.q[par], &qmap, 0, row, &sm.full[s]);
                tma_2d(sm.q[par] + QREG, &qmap, 64, row, &sm.full[s]);
            };
            auto flush = [&]() {
                griddep_wait();
                griddep_launch_dependents();
                waited = true;
                if (late_row >= 0 && elect_one()) load_q(late_row, late_stage, late_par);
                __syncwarp();
                late_row = -1;
            };
            auto draw = [&]() {   // next dynamic item, one atomic per warp
                int v = 0;
                if (lane == 0) v = sched_next(p.counters);
                return (int)gridDim.x + __shfl_sync(FULL_MASK, v, 0);
            };
            int w = blockIdx.x;
            int w_next = waited ? draw() : -1;
            while (w < total) {
                int c, g;
                sched_item(sm.ws, w, p.Hkv, b, c, g);
                const int L = sm.ws.lens[b];
                const int nch = (L + CHUNK - 1) / CHUNK;
                const int r0 = c * CHUNK;
                const int rows = min(CHUNK, L - r0);
                const int row_base = (b * p.Hkv + g) * p.max_ctx + r0;
                const int ntiles = (rows + TK - 1) / TK;
                const bool app = p.k_new != nullptr && c == nch - 1;
                const int par = item & 1;
                for (int t = 0; t < ntiles; ++t) {
                    const int nr = min(TK, rows - t * TK);
                    const bool app_tile = app && t == ntiles - 1;
                    if (!waited && (issued == STAGES || r0 + t * TK + nr == L)) flush();
                    mbar_wait(&sm.empty[stage], phase ^ 1);
                    if (t == 0) mbar_wait(&sm.q_empty[par], ((item >> 1) & 1) ^ 1);   // S of item-2 done
                    TStage &st = sm.st[stage];
                    // a tile cut short by lens is fetched in 32-row boxes: at most 31 rows
                    // past lens, not up to 127 (rows past nr are masked, their V zeroed)
                    const int nbox = nr == TK ? 0 : (nr + TAIL - 1) / TAIL;
                    uint32_t bytes = nbox ? 4u * nbox * TAIL * 128 : 4 * KREG;
                    int moff = 0;
                    uint32_t mbytes = 0;
                    const uint8_t *msrc = nullptr;
                    if (p.mask) {
                        const size_t row0 = (size_t)b * p.max_ctx;
                        const size_t j0 = row0 + sm.ws.pad[b] + r0 + t * TK;
                        const size_t a0 = j0 & ~(size_t)15;
                        size_t need = (j0 + nr - a0 + 15) & ~(size_t)15;
                        if (a0 + need > row0 + p.max_ctx) need = row0 + p.max_ctx - a0;
                        moff = (int)(j0 - a0);
                        msrc = p.mask + a0;
                        mbytes = (uint32_t)need;
                        bytes += mbytes;
                    }
                    if (t == 0) bytes += 2 * QREG;
                    if (app_tile) bytes += 2 * D * 2;
                    const int qrow = b * p.Hq + g * GS;
                    if (elect_one()) {
                        st.desc.b = b;
                        st.desc.g = g;
                        st.desc.c = c;
                        st.desc.nrows = nr;
                        st.desc.flags = (t == 0 ? F_FIRST : 0) | (t == ntiles - 1 ? F_LAST : 0) | (app_tile ? F_WRITE : 0);
                        st.desc.moff = moff;
                        st.desc.nchunks = nch;
                        st.desc.wrow = L - 1;
                        st.desc.item = item;
                        st.desc.stage = stage;
                        mbar_arrive_expect_tx(&sm.full[stage], bytes);
                        const int row = row_base + t * TK;
                        if (nbox == 0) {
                            tma_2d(st.k, &kmap, 0, row, &sm.full[stage]);
                            tma_2d(st.k + KREG, &kmap, 64, row, &sm.full[stage]);
                            tma_2d(st.v, &vmap, 0, row, &sm.full[stage]);
                            tma_2d(st.v + KREG, &vmap, 64, row, &sm.full[stage]);
                        } else {
                            for (int i = 0; i < nbox; ++i) {   // 4 KB pieces, 1024-B aligned: same swizzle
                                const uint32_t o = i * TAIL * 128;
                                tma_2d(st.k + o, &kmap32, 0, row + i * TAIL, &sm.full[stage]);
                                tma_2d(st.k + KREG + o, &kmap32, 64, row + i * TAIL, &sm.full[stage]);
                                tma_2d(st.v + o, &vmap32, 0, row + i * TAIL, &sm.full[stage]);
                                tma_2d(st.v + KREG + o, &vmap32, 64, row + i * TAIL, &sm.full[stage]);
                            }
                        }
                        if (mbytes) bulk_g2s(st.mask, msrc, mbytes, &sm.full[stage]);
                        if (app_tile) {   // always after the wait (flush above)
                            const size_t nb = ((size_t)b * p.Hkv + g) * D;
                            bulk_g2s(st.knew, p.k_new + nb, D * 2, &sm.full[stage]);
                            bulk_g2s(st.vnew, p.v_new + nb, D * 2, &sm.full[stage]);
                        }
                        if (t == 0 && waited) load_q(qrow, stage, par);
                    }
                    __syncwarp();
                    if (t == 0 && !waited) {
                        late_row = qrow;
                        late_stage = stage;
                        late_par = par;
                    }
                    ++issued;
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ++item;
                if (!waited) flush();
                if (w_next < 0) w_next = draw();
                w = w_next;
                w_next = w < total ? draw() : total;
            }
            if (!waited) flush();
            if (lane == 0) sched_done(p.counters);
            mbar_wait(&sm.empty[stage], phase ^ 1);
            if (lane == 0) {
                sm.st[stage].desc.flags = F_END;
                mbar_arrive(&sm.full[stage]);
            }
        }
    } else if (warp == 9) {
        // ============================ S issuer ============================
        // The whole warp walks the stages and waits; the tcgen05 ops go under elect.sync
        // (single UTCHMMA / UTCBAR instructions, not ptxas's per-lane loops under a
        // `lane == 0` test), lanes 0-15 patch the appended row, lane 0 writes the queues.
        {
            constexpr uint32_t idS = idesc_bf16_ab(TK, NH, 0, 0);   // A = K (K-major), B = q (K-major)
            int stage = 0;
            uint32_t phase = 0;
            int cnt[2] = {0, 0};
            while (true) {
                mbar_wait(&sm.full[stage], phase);
                TStage &st = sm.st[stage];
                const TDesc d = st.desc;
                if (d.flags & F_END) {
#pragma unroll
                    for (int g = 0; g < 2; ++g) {   // end entries for both groups and P.V issuers
                        const int n = cnt[g], sb = n & 1;
                        if (n >= 2) mbar_wait(&sm.s_free[g][sb], ((n >> 1) - 1) & 1);
                        if (lane == 0) {
                            sm.gq[g][sb].flags = F_END;
                            sm.pvq[g][n & 3].flags = F_END;
                            mbar_arrive(&sm.s_full[g][sb]);
                            mbar_arrive(&sm.s_full[g][sb]);
                        }
                    }
                    break;
                }
                const int g = d.item & 1, n = cnt[g], sb = n & 1;
                if (n >= 2) mbar_wait(&sm.s_free[g][sb], ((n >> 1) - 1) & 1);   // S(n-2) read
                if ((d.flags & F_WRITE) && lane < 16) {
                    // a2: row nrows-1 is the new token -- patch the swizzled K/V tiles
                    // the MMAs read, then the cache row (16-B chunk `lane` of each)
                    const int rr = d.nrows - 1, ch = lane;
                    const size_t dst = (((size_t)d.b * p.Hkv + d.g) * p.max_ctx + d.wrow) * D;
                    const uint4 kv = reinterpret_cast<const uint4 *>(st.knew)[ch];
                    const uint4 vv = reinterpret_cast<const uint4 *>(st.vnew)[ch];
                    *reinterpret_cast<uint4 *>(st.k + swz(rr, ch, KREG)) = kv;
                    *reinterpret_cast<uint4 *>(st.v + swz(rr, ch, KREG)) = vv;
                    reinterpret_cast<uint4 *>(p.k_w + dst)[ch] = kv;
                    reinterpret_cast<uint4 *>(p.v_w + dst)[ch] = vv;
                    fence_async_smem();
                }
                __syncwarp();
                const uint32_t ka = smem_u32(st.k), qa = smem_u32(sm.q[g]);
                const uint32_t tS = tmem + 32 * g + 16 * sb;
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)   // K = 128 dims in steps of 16
                        umma_f16(tS, smem_desc(ka + (k >> 2) * KREG + (k & 3) * 32, 16, 1024),
                                 smem_desc(qa + (k >> 2) * QREG + (k & 3) * 32, 16, 1024), idS, k > 0);
                    umma_commit(&sm.s_full[g][sb]);
                    if (d.flags & F_LAST) umma_commit(&sm.q_empty[g]);
                }
                __syncwarp();
                if (lane == 0) {
                    sm.gq[g][sb] = d;
                    sm.pvq[g][n & 3] = PvEntry{d.stage, d.flags, d.b * p.Hq + d.g * GS,
                                               (d.flags & F_LAST) && d.nchunks > 1};
                    mbar_arrive(&sm.s_full[g][sb]);            // release: the queue entries
                    if (trace && g == 0 && n < 16) tr[4 + 4 * n] = tt_now();
                }
                cnt[g] = n + 1;
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp >= 10) {
        // ============================ P.V issuer of group (warp - 10) ============================
        // whole warp waits, one elected lane issues (as the S issuer)
        {
            const int g = warp - 10;
            constexpr uint32_t idO = idesc_bf16_ab(D, NH, 1, 0);    // A = V (MN-major), B = P^T (K-major)
            const uint32_t tO = tmem + 64 + 16 * g, pa = smem_u32(sm.p[g]);
            // publish mode: a split item's ticket is released after this group's softmax
            // threads wrote its partials (pub barrier) -- deferred until the next P.V is
            // issued, so the release's wait for those writes overlaps tensor work
            int pending = -1;
            uint32_t pub_phase = 0;
            auto publish = [&]() {
                if (pending < 0) return;
                mbar_wait(&sm.pub[g], pub_phase);
                pub_phase ^= 1;
                if (lane == 0) red_add_release_gpu(p.tickets + pending, 1);
                pending = -1;
            };
            for (int n = 0;; ++n) {
                mbar_wait(&sm.p_full[g], n & 1);
                const PvEntry e = sm.pvq[g][n & 3];
                if (e.flags & F_END) {
                    publish();
                    break;
                }
                tc_fence_after();
                const uint32_t va = smem_u32(sm.st[e.stage].v);
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)   // K = 128 keys in steps of 16
                        umma_f16(tO, smem_desc(va + k * 2048, KREG, 1024),
                                 smem_desc(pa + (k >> 2) * PREG + (k & 3) * 32, 16, 1024), idO,
                                 !((e.flags & F_FIRST) && k == 0));
                    umma_commit(&sm.o_done[g]);
                    umma_commit(&sm.empty[e.stage]);
                }
                __syncwarp();
                if (trace && g == 0 && n < 16 && lane == 0) tr[7 + 4 * n] = tt_now();
                if (BATON_EXPERIMENTS && p.publish) {   // variant 23 (experiment builds)
                    publish();
                    if (e.multi) pending = e.bh0;
                }
            }
        }
    } else if (warp < 8) {
        // ============================ softmax warpgroups ============================
        const int grp = warp >> 2, wq = warp & 3;
        if (p.early) {
            griddep_wait();
            griddep_launch_dependents();
        }
        if (trace && threadIdx.x == 0) tr[2] = tt_now();
        // decode step: the previous layer's split-K merge (its partials are complete and
        // visible once griddepcontrol.wait returned), by group 1 only: group 0 starts on
        // this layer's first item at once (4 warps x 2 pairs x 148 CTAs still cover the
        // 70B shard's 1024 (slot, q head) pairs in one pass)
        if (p.prev_partial && grp == 1)
            gqa_merge_pairs(p.lens, p.prev_partial, p.prev_out, p.B, p.Hq, p.max_chunks,
                            blockIdx.x * 4 + wq, gridDim.x * 4, lane);
        if (trace && p.prev_partial && threadIdx.x == 128) tr[3] = tt_now();
        for (int b = blockIdx.x; b < p.B; b += gridDim.x) {   // empty slots -> zero rows (C6)
            if (p.lens[b] <= 0) {
                uint4 *o = reinterpret_cast<uint4 *>(p.out + (size_t)b * p.Hq * D);
                for (int i = threadIdx.x; i < p.Hq * D / 8; i += 256) o[i] = make_uint4(0, 0, 0, 0);
            }
        }
        const int r = wq * 32 + lane;                    // key row (S) / dim (O) = TMEM lane
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tO = tmem + 64 + 16 * grp;
        float m[GS], lp[GS];
        for (int n = 0;; ++n) {                          // this group's n-th tile
            const int sb = n & 1;
            mbar_wait(&sm.s_full[grp][sb], (n >> 1) & 1);
            tc_fence_after();
            const TDesc d = sm.gq[grp][sb];
            if (d.flags & F_END) {
                mbar_arrive(&sm.p_full[grp]);            // the P.V issuer reads its end entry
                break;
            }
            TStage &st = sm.st[d.stage];
            if (d.flags & F_FIRST) {
#pragma unroll
                for (int h = 0; h < GS; ++h) {
                    m[h] = -INFINITY;
                    lp[h] = 0.f;
                }
            }
            uint32_t sr[16];
            tmem_ld16(tmem + 32 * grp + 16 * sb + lane_off, sr);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&sm.s_free[grp][sb]);            // S buffer free for the MMA
            if (trace && r == 0 && grp == 0 && n < 16) tr[5 + 4 * n] = tt_now();
            bool valid = r < d.nrows;
            if (p.mask) valid = valid && st.mask[d.moff + r] != 0;
            float x[GS];
#pragma unroll
            for (int h = 0; h < GS; ++h) x[h] = valid ? __uint_as_float(sr[h]) * p.scale_log2 : -INFINITY;
            // per-head tile max: redux within the warp, then the group's 4 warps
#pragma unroll
            for (int h = 0; h < GS; ++h) {
                const int v = __reduce_max_sync(FULL_MASK, f2o(x[h]));
                if (lane == 0) sm.red[grp][sb][wq][h] = v;
            }
            named_bar_sync(1 + grp, 128);
            float alpha[GS], mref[GS];
            bool moved = false;
#pragma unroll
            for (int h = 0; h < GS; ++h) {
                int v = sm.red[grp][sb][0][h];
#pragma unroll
                for (int w2 = 1; w2 < 4; ++w2) v = max(v, sm.red[grp][sb][w2][h]);
                const float m_new = fmaxf(m[h], o2f(v));
                mref[h] = (m_new == -INFINITY) ? 0.f : m_new;
                alpha[h] = ex2(m[h] - mref[h]);
                moved = moved || (m_new != m[h]);
                m[h] = m_new;
            }
            uint16_t pb[GS];
#pragma unroll
            for (int h = 0; h < GS; ++h) {
                const __nv_bfloat16 e = __float2bfloat16_rn(ex2(x[h] - mref[h]));
                pb[h] = *reinterpret_cast<const uint16_t *>(&e);
                lp[h] = lp[h] * alpha[h] + __bfloat162float(e);
            }
            if (!valid) {   // masked / out-of-range key: its V row may hold anything
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) *reinterpret_cast<uint4 *>(st.v + swz(r, ch, KREG)) = make_uint4(0, 0, 0, 0);
            }
            // the group's P buffer and O: P.V of its previous tile must be done
            if (n > 0) mbar_wait(&sm.o_done[grp], (n - 1) & 1);
            tc_fence_after();
            if (!(d.flags & F_FIRST) && moved) {   // rescale O^T[dim r][head h] by alpha[h]
                uint32_t o[16];
                tmem_ld16(tO + lane_off, o);
                tmem_wait_ld();
#pragma unroll
                for (int h = 0; h < GS; ++h) o[h] = __float_as_uint(__uint_as_float(o[h]) * alpha[h]);
                tmem_st16(tO + lane_off, o);
                tmem_wait_st();
            }
            // P^T element (head h, key r): K-major SW128, 64 keys per 2 KB half
#pragma unroll
            for (int h = 0; h < GS; ++h) {
                const uint32_t off = (uint32_t)((r >> 6) * PREG + h * 128 + ((((r & 63) >> 3) ^ (h & 7)) << 4) + (r & 7) * 2);
                *reinterpret_cast<uint16_t *>(sm.p[grp] + off) = pb[h];
            }
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(&sm.p_full[grp]);
            if (trace && r == 0 && grp == 0 && n < 16) tr[6 + 4 * n] = tt_now();
            if (d.flags & F_LAST) {
                // ---- epilogue: wait for this tile's P.V, reduce the row sums
                mbar_wait(&sm.o_done[grp], n & 1);
                tc_fence_after();
                float lt[GS];
#pragma unroll
                for (int h = 0; h < GS; ++h) {
                    float v = lp[h];
#pragma unroll
                    for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o2);
                    if (lane == 0) sm.lsum[grp][wq][h] = v;
                }
                named_bar_sync(1 + grp, 128);
#pragma unroll
                for (int h = 0; h < GS; ++h)
                    lt[h] = sm.lsum[grp][0][h] + sm.lsum[grp][1][h] + sm.lsum[grp][2][h] + sm.lsum[grp][3][h];
                uint32_t o[16];
                tmem_ld16(tO + lane_off, o);
                tmem_wait_ld();
                tc_fence_before();
                const size_t bh0 = (size_t)d.b * p.Hq + d.g * GS;
                if (d.nchunks == 1) {
#pragma unroll
                    for (int h = 0; h < GS; ++h)
                        p.out[(bh0 + h) * D + r] = __float2bfloat16_rn(lt[h] > 0.f ? __uint_as_float(o[h]) / lt[h] : 0.f);
                } else {
#pragma unroll
                    for (int h = 0; h < GS; ++h) {
                        float *pp = p.partial + ((bh0 + h) * p.max_chunks + d.c) * (D + PREC_PAD);
                        pp[r] = __uint_as_float(o[h]);
                        if (r == 0) {
                            pp[D] = m[h];
                            pp[D + 1] = lt[h];
                        }
                    }
                    if (BATON_EXPERIMENTS && p.publish) mbar_arrive(&sm.pub[grp]);   // variant 23
                    if (p.fused) {
                        // in-kernel split-K merge: the group that draws the last ticket of
                        // (slot, kv group) merges the chunks in ascending order.  The
                        // ticket's round trip stalls this group only; the other keeps
                        // streaming.  (Group barrier, then one gpu-scope acq_rel atomic.)
                        named_bar_sync(1 + grp, 128);
                        int32_t *tk = p.tickets + bh0;
                        if (r == 0) sm.last[grp] = atom_add_acq_rel_gpu(tk, 1) == d.nchunks - 1;
                        named_bar_sync(1 + grp, 128);
                        if (sm.last[grp]) {
                            // parallel merge of the 8 heads: (A) thread (head, chunk) loads m, l;
                            // the group derives each chunk's weight f = 2^(m_c - M) in smem;
                            // (B) thread = dim accumulates all heads, 4 chunks per round trip.
                            // Chunks are taken in ascending order (batch-invariant).
                            const int nch = d.nchunks;
                            for (int i2 = r; i2 < GS * nch; i2 += 128) {
                                const int h = i2 & 7, c = i2 >> 3;
                                const float *rr = p.partial + ((bh0 + h) * p.max_chunks + c) * (D + PREC_PAD);
                                sm.mf[grp][c][h] = __ldcg(rr + D);
                                sm.ml[grp][c][h] = __ldcg(rr + D + 1);
                            }
                            named_bar_sync(1 + grp, 128);
                            float Mh[GS], Lh[GS];
#pragma unroll
                            for (int h = 0; h < GS; ++h) {
                                float Mc = -INFINITY;
                                for (int c = 0; c < nch; ++c) Mc = fmaxf(Mc, sm.mf[grp][c][h]);
                                float Lc = 0.f;
                                for (int c = 0; c < nch; ++c) {
                                    const float mc = sm.mf[grp][c][h];
                                    Lc = fmaf((mc == -INFINITY) ? 0.f : ex2(mc - Mc), sm.ml[grp][c][h], Lc);
                                }
                                Mh[h] = Mc;
                                Lh[h] = Lc;
                            }
                            float Oh[GS];
#pragma unroll
                            for (int h = 0; h < GS; ++h) Oh[h] = 0.f;
                            for (int c0 = 0; c0 < nch; c0 += 4) {
                                float ov[4][GS];
#pragma unroll
                                for (int k = 0; k < 4; ++k)
#pragma unroll
                                    for (int h = 0; h < GS; ++h)
                                        ov[k][h] = c0 + k < nch
                                                       ? __ldcg(p.partial + ((bh0 + h) * p.max_chunks + c0 + k) * (D + PREC_PAD) + r)
                                                       : 0.f;
#pragma unroll
                                for (int k = 0; k < 4; ++k)
#pragma unroll
                                    for (int h = 0; h < GS; ++h) {
                                        if (c0 + k < nch) {
                                            const float mc = sm.mf[grp][c0 + k][h];
                                            const float f = (mc == -INFINITY) ? 0.f : ex2(mc - Mh[h]);
                                            Oh[h] = fmaf(f, ov[k][h], Oh[h]);
                                        }
                                    }
                            }
#pragma unroll
                            for (int h = 0; h < GS; ++h)
                                p.out[(bh0 + h) * D + r] = __float2bfloat16_rn(Lh[h] > 0.f ? Oh[h] / Lh[h] : 0.f);
                            if (r == 0) *tk = 0;   // ready for the next launch
                        }
                    }
                }
                named_bar_sync(1 + grp, 128);   // lsum / last reused by the next item
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (trace && threadIdx.x == 0) tr[1] = tt_now();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    }
}

}  // namespace

cudaError_t launch_decode_gqa_tc(const DecodeArgs &a, cudaStream_t s, bool fused, bool publish) {
    const int num_sms = device_sms();
    const size_t smem = sizeof(TSmem) + 1024;
    {
        cudaError_t e = ensure_smem_attr(decode_gqa_tc_kernel, smem);
        if (e != cudaSuccess) return e;
    }
    if (a.dry) return cudaSuccess;
    TParams p;
    p.q = static_cast<const __nv_bfloat16 *>(a.q);
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
    p.fused = fused;
    p.prev_partial = a.prev_partial;
    p.prev_out = static_cast<__nv_bfloat16 *>(a.prev_out);
    p.publish = publish && !fused;
    if (fused && a.max_chunks > 32) return cudaErrorInvalidValue;   // see TSmem::mf
    p.B = a.slots;
    p.Hq = a.q_heads;
    p.Hkv = a.kv_heads;
    p.max_ctx = a.max_ctx;
    p.max_chunks = a.max_chunks;
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.early = a.early;
    CUtensorMap km, vm, qm, km32, vm32;
    const uint64_t dims[2] = {(uint64_t)D, (uint64_t)a.slots * a.kv_heads * a.max_ctx};
    const uint64_t strides[1] = {(uint64_t)D * 2};
    const uint32_t box[2] = {64, TK};
    const uint64_t qdims[2] = {(uint64_t)D, (uint64_t)a.slots * a.q_heads};
    const uint32_t qbox[2] = {64, NH};
    const uint32_t box32[2] = {64, TAIL};
    if (!encode_bf16_map(&km, a.k, 2, dims, strides, box) || !encode_bf16_map(&vm, a.v, 2, dims, strides, box) ||
        !encode_bf16_map(&qm, a.q, 2, qdims, strides, qbox) ||
        !encode_bf16_map(&km32, a.k, 2, dims, strides, box32) || !encode_bf16_map(&vm32, a.v, 2, dims, strides, box32))
        return cudaErrorInvalidValue;
    return launch_pdl(decode_gqa_tc_kernel, dim3(num_sms), dim3(THREADS), smem, s, km, vm, qm, km32, vm32, p);
}

}  // namespace baton

extern "C" int baton_debug_gqa_tc_trace(int on, void *host, size_t bytes) {
#if !BATON_EXPERIMENTS
    (void)on;
    (void)host;
    (void)bytes;
    return -1;   // timelines exist in experiment builds only
#endif
    if (host) {
        if (cudaMemcpyFromSymbol(host, baton::g_tt, bytes < sizeof(baton::g_tt) ? bytes : sizeof(baton::g_tt)) !=
            cudaSuccess)
            return -1;
    }
    if (on >= 0) {
        if (on) {
            static long long zero[2][baton::TT_CTAS][baton::TT_W];
            cudaMemcpyToSymbol(baton::g_tt, zero, sizeof(zero));
        }
        if (cudaMemcpyToSymbol(baton::g_tt_on, &on, sizeof(int)) != cudaSuccess) return -1;
    }
    return 0;
}
