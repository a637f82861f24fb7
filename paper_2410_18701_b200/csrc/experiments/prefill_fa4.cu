// prefill_fa4.cu -- a8 prefill attention, the FA4 layout on the 5th-gen tensor cores.
//
// EXPERIMENT BUILD ONLY (BATON_EXPERIMENTS=1, BATON_PF_KERNEL=2): passes every prefill /
// varlen / shaping parity test, but measured slower than the round-1 kernel
// (prefill_attention.cu) on every prompt shape -- DESIGN.md §6.3 has the numbers and
// the ncu reading (the softmax waits for S: S_i(j+1) can only follow PV_i(j)).
//
// What it computes ("all original queries ... are initially prefilled";
// P:L215 asynchronous P&D): causal softmax(Q K^T / sqrt(D)) V of each new prompt over
// its own tokens -- row i is the textbook SDPA of query token i over keys
// 0..i.  n prompts are packed along the token axis (varlen, cu_lens) in one launch.
//
// Why a second kernel: the round-1 kernel (prefill_attention.cu, still used for the
// shaping path's extend attention) runs one 128-row Q tile per CTA against 64-key
// tiles, two CTAs per SM.  Its S MMA (M=128, N=64) reads 6 KB of smem operands per
// 32 tensor cycles -- more than the SM's shared-memory read port -- each CTA streams
// its own copy of every K/V tile, and ncu showed its two softmax groups and the
// tensor pipe waiting on each other (56% tensor, 57% XU, 41% issue: nothing saturated).
//
// Layout here (one persistent CTA per SM; a work item = (prompt, pair of 128-row Q
// tiles, q head), heaviest first, strided over the grid):
//   * S = Q K^T with 128-key tiles: UMMA M=128, N=128, K=16 x 8 (8 KB of smem per 64
//     cycles); both Q tiles of the pair share every K/V tile (K/V smem traffic and L2
//     reads halved per FLOP);
//   * TMEM (512 columns): S0 | S1 | O0 | O1, 128 columns each.  P_i overwrites the
//     upper 64 columns of S_i as bf16 pairs and feeds O_i += P_i V as the TMEM (A)
//     operand ("TS" form);
//   * two softmax warpgroups (warps 0-3: Q tile 0, warps 4-7: Q tile 1), thread =
//     query row = TMEM lane, ping-ponged: the MMA issuer (warp 9) issues
//         S0(0) S1(0) | PV0(0) S0(1) | PV1(0) S1(1) | PV0(1) S0(2) | ...
//     so the tensor pipe runs one group's P.V and next S while the other group
//     computes its exponentials.  S_i(j+1) goes into the TMEM columns P_i(j) occupies,
//     issued after PV_i(j): the tensor pipe executes in issue order.  For the same
//     reason a softmax group that holds S_i(j+1) knows PV_i(j) is complete, so its
//     (lazy, rare) O rescale needs no extra barrier;
//   * warp 8: TMA producer -- Q tiles (2 x 32 KB), K and V tiles (32 KB each) through
//     2-stage rings, cp.async.bulk.tensor with mbarrier tx-counts.  The next work
//     item's Q and K/V stream in while this item's last tiles and epilogue run.
//   Softmax per row and 128-key tile: three tcgen05.ld round trips of 64 columns
//   (the 10-warp CTA leaves 168 registers a thread), causal -inf only on the diagonal
//   tile, the row max by 3-input FMNMX3, lazy rescale (P <= 2^rescale_t against a
//   reference max that moves only by more than rescale_t, O rescaled in TMEM on those
//   tiles), exponent FFMA2 + ex2 per key, bf16x2 packs straight into TMEM
//   (tcgen05.st x32), fp32 row sum by FADD2.  Epilogue: O_i / l -> bf16 rows.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "../common.cuh"
#include "../kernels.h"
#include "../tcgen05.cuh"
#include "../tma.h"

namespace baton {

// lazy-rescale counter (warp-tiles that rescaled O; baton_debug_prefill_rescales adds
// it to prefill_attention.cu's)
__device__ unsigned long long g_fa4_rescales = 0;

namespace {

using namespace tc;

constexpr int FM = 128;                     // rows per Q tile (UMMA M, TMEM lanes)
constexpr int FN = 128;                     // keys per K/V tile
constexpr int FD = 128;                     // head_dim
constexpr int FTHREADS = 320;               // 2 softmax warpgroups, producer warp, MMA warp
constexpr int FQ_BYTES = FM * FD * 2;       // 32 KB: two 16 KB SW128 regions (dims 0-63, 64-127)
constexpr int FQ_REG = FQ_BYTES / 2;
constexpr int FKV_BYTES = FN * FD * 2;      // 32 KB
constexpr int FKV_REG = FKV_BYTES / 2;
constexpr int F_MAXP = 64;                  // prompts per launch
constexpr int F_MAXE = 1024;                // (prompt, Q-tile pair) entries per launch

struct __align__(1024) FaSmem {
    uint8_t q[2][FQ_BYTES];
    uint8_t k[2][FKV_BYTES];
    uint8_t v[2][FKV_BYTES];
    uint64_t q_full[2], q_empty[2], k_full[2], k_empty[2], v_full[2], v_empty[2];
    uint64_t s_full[2], p_full[2], o_done[2], o_free[2];
    uint32_t tmem_base;
};

struct FaParams {
    int Hq, Hkv, n_work, total;
    float scale_log2, rescale_t;
    __nv_bfloat16 *out;
    int32_t start[F_MAXP], len[F_MAXP];
    uint32_t entry[F_MAXE];                 // prompt << 16 | pair, heaviest first
};

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
BATON_DEV float2 fadd2(float2 a, float2 b) {
    uint64_t A, B, D;
    asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    float2 d;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(D));
    return d;
}
BATON_DEV float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// one work item: prompt, the pair's first row, q head, key tiles of each Q tile
struct Work {
    int s0, len, q0, h, n0, n1;
    bool has1;
};
BATON_DEV Work decode_work(const FaParams &p, int w) {
    Work k;
    const uint32_t e = p.entry[w / p.Hq];
    const int pi = (int)(e >> 16);
    k.h = w % p.Hq;
    k.s0 = p.start[pi];
    k.len = p.len[pi];
    k.q0 = (int)(e & 0xffff) * 2 * FM;
    k.has1 = k.q0 + FM < k.len;
    k.n0 = k.q0 / FN + 1;                   // keys [0, q0 + 128): up to the diagonal
    k.n1 = k.has1 ? k.n0 + 1 : 0;
    return k;
}

// 10 warps: SM sub-partitions 0/1 hold 3 of them, so at most 16384 / 96 = 170 registers
__global__ void __launch_bounds__(FTHREADS, 1)
prefill_fa4_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const FaParams p) {
    extern __shared__ uint8_t smem_raw[];
    FaSmem &sm = *reinterpret_cast<FaSmem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.q_full[s], 1);
            mbar_init(&sm.q_empty[s], 1);
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.k_empty[s], 1);
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.v_empty[s], 1);
            mbar_init(&sm.s_full[s], 1);
            mbar_init(&sm.p_full[s], 128);
            mbar_init(&sm.o_done[s], 1);
            mbar_init(&sm.o_free[s], 128);
        }
        fence_mbar_init();
    }
    if (warp == 0) {   // TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 8) {
        // ======================= TMA producer =======================
        if (lane == 0) {
            prefetch_tmap(&tm_q);
            prefetch_tmap(&tm_k);
            prefetch_tmap(&tm_v);
            int nq[2] = {0, 0}, kc = 0;
            for (int w = blockIdx.x; w < p.n_work; w += gridDim.x) {
                const Work wk = decode_work(p, w);
                const int g = wk.h * p.Hkv / p.Hq;
                for (int i = 0; i < 2; ++i) {
                    if (i == 1 && !wk.has1) break;
                    if (nq[i] > 0) mbar_wait(&sm.q_empty[i], (nq[i] - 1) & 1);   // last tile's S MMAs done
                    ++nq[i];
                    mbar_arrive_expect_tx(&sm.q_full[i], FQ_BYTES);
                    const int row = wk.s0 + wk.q0 + i * FM;
                    tma_load_3d(sm.q[i], &tm_q, 0, row, wk.h, &sm.q_full[i]);
                    tma_load_3d(sm.q[i] + FQ_REG, &tm_q, 64, row, wk.h, &sm.q_full[i]);
                }
                const int nk = wk.has1 ? wk.n1 : wk.n0;
                for (int j = 0; j < nk; ++j, ++kc) {
                    const int s = kc & 1, u = kc >> 1;
                    const int row = wk.s0 + j * FN;
                    if (u > 0) mbar_wait(&sm.k_empty[s], (u - 1) & 1);
                    mbar_arrive_expect_tx(&sm.k_full[s], FKV_BYTES);
                    tma_load_3d(sm.k[s], &tm_k, 0, row, g, &sm.k_full[s]);
                    tma_load_3d(sm.k[s] + FKV_REG, &tm_k, 64, row, g, &sm.k_full[s]);
                    if (u > 0) mbar_wait(&sm.v_empty[s], (u - 1) & 1);
                    mbar_arrive_expect_tx(&sm.v_full[s], FKV_BYTES);
                    tma_load_3d(sm.v[s], &tm_v, 0, row, g, &sm.v_full[s]);
                    tma_load_3d(sm.v[s] + FKV_REG, &tm_v, 64, row, g, &sm.v_full[s]);
                }
            }
        }
    } else if (warp == 9) {
        // ======================= MMA issuer =======================
        // whole warp: decisions from lane 0's barrier polls broadcast to every lane, the
        // tcgen05 ops under elect.sync (round 2; under `lane == 0` ptxas wrapped each one
        // in a per-lane ELECT loop)
        {
            constexpr uint32_t idS = idesc_bf16(FM, FN, 0);   // B = K tile, K-major
            constexpr uint32_t idO = idesc_bf16(FM, FD, 1);   // A = P (TMEM), B = V tile, MN-major
            int nq[2] = {0, 0}, np[2] = {0, 0}, kc = 0;
            // S_i(j) = Q_i K(j)^T into TMEM columns 128 i; after the tile's last S_i, Q_i's
            // smem may take the next work item's Q tile
            auto issue_s = [&](int i, int j, int ni) {
                const int s = (kc + j) & 1;
                const uint32_t qa = smem_u32(sm.q[i]), ka = smem_u32(sm.k[s]);
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)        // K = head_dim in steps of 16 (32 B)
                        umma_f16(tmem + 128 * i, smem_desc(qa + (k >> 2) * FQ_REG + (k & 3) * 32, 16, 1024),
                                 smem_desc(ka + (k >> 2) * FKV_REG + (k & 3) * 32, 16, 1024), idS, k > 0);
                    umma_commit(&sm.s_full[i]);
                    if (j == ni - 1) umma_commit(&sm.q_empty[i]);
                }
                __syncwarp();
            };
            auto issue_pv = [&](int i, int j) {    // O_i += P_i(j) V(j)
                const int s = (kc + j) & 1;
                const uint32_t va = smem_u32(sm.v[s]);
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)        // K = 128 keys in steps of 16 (8 TMEM columns of bf16 pairs)
                        umma_f16_ts(tmem + 256 + 128 * i, tmem + 128 * i + 64 + 8 * k,
                                    smem_desc(va + k * 2048, FKV_REG, 1024), idO, (j > 0 || k > 0));
                }
                __syncwarp();
            };
            auto commit = [&](uint64_t *bar) {
                if (elect_one()) umma_commit(bar);
                __syncwarp();
            };
            auto wait_k = [&](int j) {
                const int t = kc + j;
                mbar_wait(&sm.k_full[t & 1], (t >> 1) & 1);
                tc_fence_after();
            };
            // Event-driven: P.V (and the next S) of whichever group published its P
            // first -- a strict 0,1,0,1 order would hold one group's MMAs behind the
            // other group's softmax.  K(j) / V(j) are released once every group that
            // uses them issued its S(j) / P.V(j).
            for (int w = blockIdx.x; w < p.n_work; w += gridDim.x) {
                const Work wk = decode_work(p, w);
                const int nk = wk.has1 ? wk.n1 : wk.n0;
                const int n[2] = {wk.n0, wk.n1};
                mbar_wait(&sm.q_full[0], nq[0] & 1);
                if (wk.has1) mbar_wait(&sm.q_full[1], nq[1] & 1);
                wait_k(0);
                issue_s(0, 0, wk.n0);
                if (wk.has1) issue_s(1, 0, wk.n1);
                commit(&sm.k_empty[kc & 1]);
                int next[2] = {0, wk.has1 ? 0 : n[1]};     // next P.V per group
                int k_ready = 0, v_ready = -1;              // K(<= k_ready), V(<= v_ready) waited
                int s_cnt[4] = {0, 0, 0, 0}, v_cnt[4] = {0, 0, 0, 0};   // per j & 3: S / P.V issued
                int last = 1;
                while (next[0] < n[0] || next[1] < n[1]) {
                    // a group is ready when its P is published and the V / next K tile it
                    // needs are loaded (never block here: one group may be a tile ahead, and
                    // the stage it needs frees only when the other group moves on)
                    auto ready = [&](int c) {
                        if (next[c] >= n[c] || !mbar_test_wait(&sm.p_full[c], np[c] & 1)) return false;
                        const int j = next[c];
                        if (j > v_ready && !mbar_test_wait(&sm.v_full[(kc + j) & 1], ((kc + j) >> 1) & 1))
                            return false;
                        if (j + 1 < n[c] && j + 1 > k_ready &&
                            !mbar_test_wait(&sm.k_full[(kc + j + 1) & 1], ((kc + j + 1) >> 1) & 1))
                            return false;
                        return true;
                    };
                    int i = -1;
                    if (lane == 0)
                        for (int t = 1; t <= 2 && i < 0; ++t) {   // round robin over ready groups
                            const int c = (last + t) & 1;
                            if (ready(c)) i = c;
                        }
                    i = __shfl_sync(FULL_MASK, i, 0);   // one decision for the whole warp
                    if (i < 0) continue;                     // spin (test_wait does not suspend)
                    last = i;
                    const int j = next[i]++;
                    ++np[i];
                    if (j == 0 && nq[i] > 0) mbar_wait(&sm.o_free[i], (nq[i] - 1) & 1);   // epilogue read O_i
                    if (j > v_ready) {
                        const int t = kc + j;
                        mbar_wait(&sm.v_full[t & 1], (t >> 1) & 1);
                        v_ready = j;
                    }
                    tc_fence_after();
                    issue_pv(i, j);
                    if (j == n[i] - 1) commit(&sm.o_done[i]);
                    const int v_need = (j < n[0]) + (j < n[1]);
                    if (++v_cnt[j & 3] == v_need) {          // V(j) consumed by every group
                        v_cnt[j & 3] = 0;
                        commit(&sm.v_empty[(kc + j) & 1]);
                    }
                    if (j + 1 < n[i]) {
                        if (j + 1 > k_ready) {
                            wait_k(j + 1);
                            k_ready = j + 1;
                        }
                        issue_s(i, j + 1, n[i]);
                        const int k_need = (j + 1 < n[0]) + (j + 1 < n[1]);
                        if (++s_cnt[(j + 1) & 3] == k_need) {   // K(j+1) consumed
                            s_cnt[(j + 1) & 3] = 0;
                            commit(&sm.k_empty[(kc + j + 1) & 1]);
                        }
                    }
                }
                ++nq[0];
                if (wk.has1) ++nq[1];
                kc += nk;
            }
        }
    } else {
        // ======================= softmax warpgroups =======================
        const int grp = warp >> 2;                       // Q tile of the pair
        const int row = (warp & 3) * 32 + lane;          // query row within the tile = TMEM lane
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + 128 * grp + lane_off, tO = tmem + 256 + 128 * grp + lane_off;
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        int ns = 0, nt = 0;                              // S tiles / work items of this group
        for (int w = blockIdx.x; w < p.n_work; w += gridDim.x) {
            const Work wk = decode_work(p, w);
            if (grp == 1 && !wk.has1) continue;
            const int n = grp == 0 ? wk.n0 : wk.n1;
            const int qi = wk.q0 + grp * FM + row;       // query row within the prompt
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < n; ++j, ++ns) {
                mbar_wait(&sm.s_full[grp], ns & 1);
                tc_fence_after();
                // The S row in TMEM is read 64 columns per tcgen05.ld round trip (at most 64
                // scores + 32 packed P live in registers).  P (key 2c in the low half of
                // column 64 + c) only overwrites scores already in registers: keys 64-127
                // go first (-> P columns 96-127), then keys 0-63 (-> P columns 64-95).
                // Diagonal tile: keys c > lim causally masked (-inf).
                //   fast path (the reference max m is set): exponentials against m while
                //   the chunk max is checked; a chunk whose max exceeds m + rescale_t in
                //   any lane of the warp moves the reference (keys 64-127: nothing stored
                //   yet, recompute; keys 0-63: also rescale the stored P of 64-127);
                //   first tile of a work item: the row max first (two passes).
                const bool diag = j == n - 1;
                const int lim = qi - j * FN;
                uint32_t ra[32], rb[32];
                auto load2 = [&](int c0) {
                    tmem_ld32(tS + c0, ra);
                    tmem_ld32(tS + c0 + 32, rb);
                    tmem_wait_ld();
                    if (diag) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            if (c0 + i > lim) ra[i] = __float_as_uint(-INFINITY);
                            if (c0 + 32 + i > lim) rb[i] = __float_as_uint(-INFINITY);
                        }
                    }
                };
                auto max2 = [&](float acc) {
                    float a0 = acc, a1 = -INFINITY;
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {   // 3-input FMNMX3, two chains
                        a0 = fmax3(a0, __uint_as_float(ra[i]), __uint_as_float(ra[i + 1]));
                        a1 = fmax3(a1, __uint_as_float(rb[i]), __uint_as_float(rb[i + 1]));
                    }
                    return fmaxf(a0, a1);
                };
                auto pack2 = [&](uint32_t (&pk)[32], float mref, float2 &rs2) {
                    const float2 nr2 = make_float2(-mref, -mref);
#pragma unroll
                    for (int i = 0; i < 64; i += 2) {
                        const uint32_t x0 = i < 32 ? ra[i] : rb[i - 32], x1 = i < 32 ? ra[i + 1] : rb[i - 31];
                        float2 a = ffma2(make_float2(__uint_as_float(x0), __uint_as_float(x1)), sc2, nr2);
                        a.x = ex2(a.x);
                        a.y = ex2(a.y);
                        const __nv_bfloat162 b = __floats2bfloat162_rn(a.x, a.y);
                        rs2 = fadd2(rs2, a);
                        pk[i / 2] = *reinterpret_cast<const uint32_t *>(&b);
                    }
                };
                // the new reference for a chunk max mx (log2 units): moves only past m + t
                auto move_ref = [&](float mx) {
                    return (mx > m + p.rescale_t || m == -INFINITY) ? fmaxf(m, mx) : m;
                };
                float alpha = 1.f;                       // O and l scale of this tile
                float2 rs2 = make_float2(0.f, 0.f);
                float mref = m;
                if (m == -INFINITY) {                    // first tile: the row max first
                    load2(0);
                    float mx = max2(-INFINITY);
                    load2(64);
                    mx = max2(mx) * p.scale_log2;        // -inf stays -inf
                    const float m_new = move_ref(mx);
                    mref = (m_new == -INFINITY) ? 0.f : m_new;   // keeps exp2 finite
                    alpha = ex2(m - mref);
                    m = m_new;
                    uint32_t pk[32];
                    pack2(pk, mref, rs2);                // keys 64-127
                    tmem_st32(tS + 96, pk);
                } else {
                    load2(64);
                    uint32_t pk[32];
                    pack2(pk, mref, rs2);                // keys 64-127 against m
                    const float mx = max2(-INFINITY) * p.scale_log2;
                    if (__any_sync(FULL_MASK, mx > m + p.rescale_t)) {
                        const float m_new = move_ref(mx);
                        mref = m_new;
                        alpha = ex2(m - mref);
                        m = m_new;
                        rs2 = make_float2(0.f, 0.f);
                        pack2(pk, mref, rs2);            // recompute against the new reference
                    }
                    tmem_st32(tS + 96, pk);
                }
                load2(0);
                {
                    uint32_t pk[32];
                    const float mref0 = mref;
                    pack2(pk, mref, rs2);                // keys 0-63
                    const float mx = max2(-INFINITY) * p.scale_log2;
                    if (__any_sync(FULL_MASK, mx > m + p.rescale_t)) {
                        // the reference moves after keys 64-127 were stored: rescale them
                        const float m_new = move_ref(mx);
                        const float f = ex2(mref0 - m_new);   // 1 in the lanes that keep m
                        mref = m_new;
                        alpha *= f;
                        m = m_new;
                        rs2 = make_float2(rs2.x * 0.f, rs2.y * 0.f);
                        {
                            uint32_t ph[32];
                            tmem_ld32(tS + 96, ph);
                            tmem_wait_ld();
                            float2 r2 = make_float2(0.f, 0.f);
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162 *>(&ph[i]);
                                float2 v = __bfloat1622float2(b);
                                v.x *= f;
                                v.y *= f;
                                r2 = fadd2(r2, v);
                                b = __floats2bfloat162_rn(v.x, v.y);
                                ph[i] = *reinterpret_cast<const uint32_t *>(&b);
                            }
                            tmem_st32(tS + 96, ph);
                            rs2 = r2;                    // keys 64-127 (bf16-rounded sums)
                        }
                        pack2(pk, mref, rs2);            // keys 0-63 against the new reference
                    }
                    tmem_st32(tS + 64, pk);
                }
                l = l * alpha + (rs2.x + rs2.y);
                // O_grp rescale: holding S(j) means PV(j-1) is complete (issued before S(j))
                if (j > 0 && __any_sync(FULL_MASK, alpha != 1.f)) {
                    if (lane == 0) atomicAdd(&g_fa4_rescales, 1ull);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + 32 * c, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                        tmem_st32(tO + 32 * c, o);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&sm.p_full[grp]);
            }
            // epilogue: O / l -> bf16 once the tile's last P.V is done
            mbar_wait(&sm.o_done[grp], nt & 1);
            tc_fence_after();
            const float inv = l > 0.f ? 1.f / l : 0.f;
            __nv_bfloat16 *orow = p.out + ((size_t)wk.h * p.total + wk.s0 + qi) * FD;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + 32 * c, o);
                tmem_wait_ld();
                if (qi < wk.len) {
                    uint32_t wv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(o[2 * i]) * inv,
                                                                       __uint_as_float(o[2 * i + 1]) * inv);
                        wv[i] = *reinterpret_cast<const uint32_t *>(&b);
                    }
                    uint4 *o4 = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                    for (int i = 0; i < 4; ++i) o4[i] = make_uint4(wv[4 * i], wv[4 * i + 1], wv[4 * i + 2], wv[4 * i + 3]);
                }
            }
            tc_fence_before();
            mbar_arrive(&sm.o_free[grp]);                // O_grp may be overwritten
            ++nt;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

bool make_map3(CUtensorMap *m, const void *base, int heads, int rows, int box_rows) {
    const uint64_t dims[3] = {(uint64_t)FD, (uint64_t)rows, (uint64_t)heads};
    const uint64_t strides[2] = {(uint64_t)FD * 2, (uint64_t)rows * FD * 2};
    const uint32_t box[3] = {64, (uint32_t)box_rows, 1};
    return encode_bf16_map(m, base, 3, dims, strides, box);
}

}  // namespace

long long fa4_rescale_count(bool reset) {
    unsigned long long v = 0;
    if (cudaMemcpyFromSymbol(&v, g_fa4_rescales, sizeof(v)) != cudaSuccess) return -1;
    if (reset) {
        const unsigned long long z = 0;
        if (cudaMemcpyToSymbol(g_fa4_rescales, &z, sizeof(z)) != cudaSuccess) return -1;
    }
    return (long long)v;
}

cudaError_t launch_prefill_fa4_varlen(const void *q, const void *k, const void *v, void *out,
                                      const int32_t *cu_lens, int n, int q_heads, int kv_heads,
                                      float scale, float rescale_t, cudaStream_t s) {
    if (n < 1 || n > F_MAXP || cu_lens[0] != 0) return cudaErrorInvalidValue;
    FaParams p{};
    int ne = 0;
    for (int i = 0; i < n; ++i) {
        const int len = cu_lens[i + 1] - cu_lens[i];
        if (len < 1) return cudaErrorInvalidValue;
        p.start[i] = cu_lens[i];
        p.len[i] = len;
        const int npair = (len + 2 * FM - 1) / (2 * FM);
        if (ne + npair > F_MAXE || npair > 0xffff) return cudaErrorInvalidValue;
        for (int t = 0; t < npair; ++t) p.entry[ne++] = ((uint32_t)i << 16) | (uint32_t)t;
    }
    // heaviest first (K/V tiles of the pair), ties by prompt then pair
    auto cost = [&](uint32_t e) {
        const int len = p.len[e >> 16], q0 = (int)(e & 0xffff) * 2 * FM;
        return (std::min(q0 + 2 * FM, len) + FN - 1) / FN;
    };
    std::stable_sort(p.entry, p.entry + ne, [&](uint32_t a, uint32_t b) { return cost(a) > cost(b); });
    const int total = cu_lens[n];
    CUtensorMap mq, mk, mv;
    if (!make_map3(&mq, q, q_heads, total, FM) || !make_map3(&mk, k, kv_heads, total, FN) ||
        !make_map3(&mv, v, kv_heads, total, FN))
        return cudaErrorInvalidValue;
    p.Hq = q_heads;
    p.Hkv = kv_heads;
    p.n_work = ne * q_heads;
    p.total = total;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.rescale_t = rescale_t;
    p.out = static_cast<__nv_bfloat16 *>(out);
    const size_t smem = sizeof(FaSmem) + 1024;
    cudaError_t e = ensure_smem_attr(prefill_fa4_kernel, smem);
    if (e != cudaSuccess) return e;
    const int grid = std::min(device_sms(), p.n_work);
    prefill_fa4_kernel<<<grid, FTHREADS, smem, s>>>(mq, mk, mv, p);
    return cudaGetLastError();
}

}  // namespace baton
