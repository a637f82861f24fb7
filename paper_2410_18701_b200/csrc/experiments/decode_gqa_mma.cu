// decode_gqa.cu -- a3 for grouped-query attention (configs[3]: 64 q heads / 8 kv
// heads): the group of q heads that share a kv head forms a real dense tile, so
// the dot products and the P.V product run on the tensor cores (mma.sync
// m16n8k16 bf16 -> fp32), while K/V are still streamed from HBM exactly once.
//
//   work item = (slot b, kv head g, 256-key chunk c); GS = q_heads/kv_heads = 8
//   producer (one elected lane): each 64-key K/V tile arrives by TMA 2-D tensor
//     loads (4 boxes of 64 rows x 64 dims, SWIZZLE_128B: 16-B chunk c of row r of
//     half h lands at h*TILE*128 + r*128 + ((c ^ r) & 7)*16) so every ldmatrix below
//     is bank-conflict free; q and the tile's mask bytes by 1-D bulk copies; all
//     completion tracked by one mbarrier tx-count.  A box may extend past lens in
//     the last tile of a slot: those rows are masked and their V zeroed, never used.
//     (A single warp's cp.async stream was measured at 1.3 TB/s -- too few bytes
//     in flight; the TMA engine keeps 4 x 32 KB per SM in flight.)
//   consumer warps (16 keys each): S[16 x 16keys] = Q[16(8 real heads) x 128] K^T
//     (16 MMAs), masked online softmax per head row (quad shuffles), P kept in
//     registers as the A fragment of O[16 x 128] += P V (16 MMAs, V via
//     ldmatrix.trans).
//   fused append (a2): the tile holding row lens-1 also brings the new token's k/v
//     (bulk copies into the stage's side buffer); the warp owning that row patches
//     it into the swizzled tile and writes it to the cache row.
//   epilogue: 4 warp states merged in smem; single chunk -> bf16 out, else an fp32
//     split-K partial (same workspace layout as decode_attention.cu); no tickets,
//     no fences: decode_combine_kernel, PDL-chained behind this launch, merges the
//     chunks in ascending order.  The combine triggers its dependents right after
//     its own wait, so the NEXT layer's launch (p.early) streams its first K/V ring
//     while the combine runs.  (An in-kernel last-arriver merge was measured: the
//     gpu-scope release/acquire and the 14-chunk merges of one warp left the grid
//     open ~8 us after the streaming ended -- profiles/r01_gqa_fused.md.)
//
// EXPERIMENT BUILD ONLY (BATON_EXPERIMENTS=1): the round-1 mma.sync GQA kernel,
// kept for A/B runs against the tcgen05 default (profiles/r01_gqa_engine_sweep.md).
#include <cstdlib>

#include "../common.cuh"
#include "../kernels.h"
#include "../sched.cuh"
#include "../tma.h"

namespace baton {


// Debug timeline (off unless baton_debug_gqa_trace(1, ...) was called): per CTA,
// [0] enter [1] work list built [2] exit [3] items [4] smid, then per item k
// [8+4k] item w, [9+4k] first TMA issued, [10+4k] first tile ready, [11+4k] epilogue
// done (k < 8), [40+2t] tile t wait start, [41+2t] tile t ready (bit 62: it was
// already complete when the wait began), t < 12.
// Launch l writes slot l % TRACE_L (host launch counter, baked into captured graphs).
constexpr int TRACE_L = 8, TRACE_CTAS = 256, TRACE_W = 64;
__device__ int g_trace_on;
__device__ long long g_trace[TRACE_L][TRACE_CTAS][TRACE_W];
static int g_trace_launch = 0;
BATON_DEV long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

namespace {

constexpr int D = 128;
constexpr int GS = 8;                       // q heads per kv head
// CW (consumer warps), KP (keys per consumer warp per tile: 16 or 32, i.e. one or
// two independent 16-key MMA chains), STAGES and CTAs/SM are template parameters; a
// tile has TILE = CW * KP keys and its two 64-dim halves are HALF = TILE * 128 bytes.
constexpr int F_FIRST = 1, F_LAST = 2, F_END = 4, F_WRITE = 8;
constexpr int QROW = D + 8;                 // q row stride in smem (272 B: rows 4 banks apart)

struct Desc {
    int32_t b, g, c, nrows, flags, moff, nchunks, wrow;
};

template <int CW, int KP>
struct __align__(1024) Stage {
    static constexpr int TILE = CW * KP;
    static constexpr int HALF = TILE * 128;
    uint8_t k[2 * HALF];
    uint8_t v[2 * HALF];
    __nv_bfloat16 q[GS * QROW];             // 8 head rows, padded: conflict-free fragment loads
    __nv_bfloat16 knew[D], vnew[D];         // appended row (F_WRITE tiles)
    uint8_t mask[TILE + 16];
    Desc desc;
};

template <int CW, int KP, int STAGES, int RB>
struct Smem {
    Stage<CW, KP> st[STAGES];
    uint64_t full[STAGES], empty[STAGES];
    WorkSched ws;
    alignas(16) float red_o[RB][CW][GS][D + 4];    // +4: the 8 head rows 4 banks apart
    float red_m[RB][CW][GS], red_l[RB][CW][GS];
};

struct Params {
    const __nv_bfloat16 *q, *k, *v;
    const __nv_bfloat16 *k_new, *v_new;     // fused append (nullable)
    __nv_bfloat16 *k_w, *v_w;               // cache base for the append write-back
    int32_t *counters;
    const uint8_t *mask;
    const int32_t *lens, *pad;
    __nv_bfloat16 *out;
    float *partial;
    int32_t *tickets;
    int B, Hq, Hkv, max_ctx, max_chunks;
    float scale_log2;
    bool early;                             // prefetch before griddepcontrol.wait
    int trace_slot;                         // debug timeline slot
};

BATON_DEV uint32_t swz(int row, int chunk, int half) {   // byte offset of 16-B chunk (0..15) of a row
    return (uint32_t)((chunk >> 3) * half + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
}
BATON_DEV void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
BATON_DEV void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
BATON_DEV void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                        uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
BATON_DEV uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&b);
}

BATON_DEV void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <int CW, int KP, int STAGES, int RB, int MINB>
__global__ void __launch_bounds__((CW + 1) * 32, MINB)
decode_gqa_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                  const Params p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for the SWIZZLE_128B boxes; offsetting the __shared__ array
    // itself keeps the shared address space visible to the compiler (LDS, not LD)
    constexpr int TILE = CW * KP, HALF = TILE * 128, NG = KP / 16;
    static_assert(KP % 16 == 0 && TILE <= 256, "tile shape");
    Smem<CW, KP, STAGES, RB> &sm =
        *reinterpret_cast<Smem<CW, KP, STAGES, RB> *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool trace = g_trace_on && blockIdx.x < TRACE_CTAS;
    long long *tr = g_trace[p.trace_slot][trace ? blockIdx.x : 0];
    if (trace && threadIdx.x == 0) {
        tr[0] = gtimer();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        tr[4] = smid;
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&sm.full[s], 1);       // producer's arrive.expect_tx (+ TMA bytes)
            mbar_init(&sm.empty[s], CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // PDL, as in decode_attention.cu: with p.early the producer builds the work list
    // and issues the first ring of K/V boxes (never the tile holding row lens-1) of a
    // statically assigned first item before the wait; q, k_new and all writes after.
    if (!p.early) {
        griddep_wait();
        griddep_launch_dependents();
    }

    if (warp == CW) {
        // ============================ producer warp ============================
        sched_build(sm.ws, p.lens, p.pad, p.B, p.Hkv, lane);
        if (lane != 0) return;
        if (trace) tr[1] = gtimer();
        int titem = 0;
        const int total = sched_total(sm.ws, p.Hkv);
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
            if (late_q)
                for (int hq = 0; hq < GS; ++hq)
                    bulk_g2s(sm.st[late_stage].q + hq * QROW, late_q + hq * D, D * 2, &sm.full[late_stage]);
            late_q = nullptr;
        };
        int w = blockIdx.x;   // static first item; the rest from the dynamic counter
        int w_next = waited ? (int)gridDim.x + sched_next(p.counters) : -1;
        while (w < total) {
            int c, g;
            sched_item(sm.ws, w, p.Hkv, b, c, g);
            const int L = sm.ws.lens[b];
            const int nch = (L + CHUNK - 1) / CHUNK;
            const int r0 = c * CHUNK;
            const int rows = min(CHUNK, L - r0);
            const int row_base = (b * p.Hkv + g) * p.max_ctx + r0;   // row in the 2-D tensor map
            const int ntiles = (rows + TILE - 1) / TILE;
            const bool app = p.k_new != nullptr && c == nch - 1;
            if (trace && titem < 8) {
                tr[8 + 4 * titem] = w;
                tr[9 + 4 * titem] = gtimer();
            }
            ++titem;
            for (int t = 0; t < ntiles; ++t) {
                const int nr = min(TILE, rows - t * TILE);
                const bool app_tile = app && t == ntiles - 1;
                // row L-1 may still be written by the previous (same-layer) kernel
                if (!waited && (issued == STAGES || r0 + t * TILE + nr == L)) flush();
                mbar_wait(&sm.empty[stage], phase ^ 1);
                Stage<CW, KP> &st = sm.st[stage];
                uint32_t bytes = 4 * HALF;      // full boxes, OOB rows zero-filled
                int moff = 0;
                uint32_t mbytes = 0;
                const uint8_t *msrc = nullptr;
                if (p.mask) {
                    const size_t row0 = (size_t)b * p.max_ctx;
                    const size_t j0 = row0 + sm.ws.pad[b] + r0 + t * TILE;
                    const size_t a0 = j0 & ~(size_t)15;
                    size_t need = (j0 + nr - a0 + 15) & ~(size_t)15;
                    if (a0 + need > row0 + p.max_ctx) need = row0 + p.max_ctx - a0;
                    moff = (int)(j0 - a0);
                    msrc = p.mask + a0;
                    mbytes = (uint32_t)need;
                    bytes += mbytes;
                }
                if (t == 0) bytes += GS * D * 2;
                if (app_tile) bytes += 2 * D * 2;
                st.desc.b = b;
                st.desc.g = g;
                st.desc.c = c;
                st.desc.nrows = nr;
                st.desc.flags = (t == 0 ? F_FIRST : 0) | (t == ntiles - 1 ? F_LAST : 0) | (app_tile ? F_WRITE : 0);
                st.desc.moff = moff;
                st.desc.nchunks = nch;
                st.desc.wrow = L - 1;
                mbar_arrive_expect_tx(&sm.full[stage], bytes);
                const int row = row_base + t * TILE;
                tma_load_2d(st.k, &kmap, 0, row, &sm.full[stage]);
                tma_load_2d(st.k + HALF, &kmap, 64, row, &sm.full[stage]);
                tma_load_2d(st.v, &vmap, 0, row, &sm.full[stage]);
                tma_load_2d(st.v + HALF, &vmap, 64, row, &sm.full[stage]);
                if (mbytes) bulk_g2s(st.mask, msrc, mbytes, &sm.full[stage]);
                if (app_tile) {   // (always after the wait: see the flush above)
                    const size_t nb = ((size_t)b * p.Hkv + g) * D;
                    bulk_g2s(st.knew, p.k_new + nb, D * 2, &sm.full[stage]);
                    bulk_g2s(st.vnew, p.v_new + nb, D * 2, &sm.full[stage]);
                }
                if (t == 0) {   // the group's 8 query rows (contiguous 2 KB)
                    const __nv_bfloat16 *qsrc = p.q + ((size_t)b * p.Hq + g * GS) * D;
                    if (waited) {
                        for (int hq = 0; hq < GS; ++hq)
                            bulk_g2s(st.q + hq * QROW, qsrc + hq * D, D * 2, &sm.full[stage]);
                    } else {
                        late_q = qsrc;
                        late_stage = stage;
                    }
                }
                ++issued;
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (!waited) flush();
            if (w_next < 0) w_next = (int)gridDim.x + sched_next(p.counters);
            w = w_next;
            w_next = w < total ? (int)gridDim.x + sched_next(p.counters) : total;
        }
        if (!waited) flush();
        sched_done(p.counters);
        mbar_wait(&sm.empty[stage], phase ^ 1);
        sm.st[stage].desc.flags = F_END;
        mbar_arrive(&sm.full[stage]);
        return;
    }

    // ============================ consumer warps ============================
    if (p.early) {
        griddep_wait();
        griddep_launch_dependents();
    }
    for (int b = blockIdx.x; b < p.B; b += gridDim.x) {   // empty slots -> zero rows (C6)
        if (p.lens[b] <= 0) {
            uint4 *o = reinterpret_cast<uint4 *>(p.out + (size_t)b * p.Hq * D);
            for (int i = threadIdx.x; i < p.Hq * D / 8; i += CW * 32) o[i] = make_uint4(0, 0, 0, 0);
        }
    }
    // Transposed formulation (keys and dims as the MMA's M so no row is padding):
    //   S^T[16 keys x 8 heads]  = K[16 x 128] . Q^T            (8 MMAs per tile)
    //   O^T[128 dims x 8 heads] += V^T[128 x 16 keys] . P^T     (8 MMAs per tile)
    const int r4 = lane >> 2;            // fragment row group
    const int c2 = (lane & 3) * 2;       // fragment column pair (heads c2, c2+1 in C)
    uint32_t qb[8][2];                   // Q^T B-fragments: head r4, dims 16k + c2 (+8)
    float o[8][4];                       // O^T: dims 16mt + r4 (+8) x heads c2, c2+1
    float m[2], l[2];                    // softmax state of heads c2, c2+1
    int stage = 0;
    uint32_t phase = 0;
    int rb = 0;                          // merge buffer of the current item
    int citem = 0, ctile = 0;
    while (true) {
        long long t_w = 0;
        bool was_ready = false;
        if (trace && threadIdx.x == 0) {
            t_w = gtimer();
            was_ready = mbar_test_wait(&sm.full[stage], phase);
        }
        mbar_wait(&sm.full[stage], phase);
        Stage<CW, KP> &st = sm.st[stage];
        const Desc d = st.desc;
        if (d.flags & F_END) break;
        if (trace && threadIdx.x == 0 && (d.flags & F_FIRST) && citem < 8)
            tr[10 + 4 * citem] = gtimer();
        if (trace && threadIdx.x == 0 && ctile < 4) {
            tr[40 + 2 * ctile] = t_w;
            tr[41 + 2 * ctile] = gtimer() | (was_ready ? (1LL << 62) : 0);
        }
        ++ctile;
        // phase clocks of warp 0 on its 3rd tile (debug): [48] start [49] S done
        // [50] softmax done [51] P fragments done [52] P.V done [53] released
        const bool ph = trace && warp == 0 && ctile == 3;
        auto phase_clock = [&](int slot, float dep) {
            if (ph) {
                if (__float_as_uint(dep) == 0x7fc00001u) tr[63] = 1;   // wait for dep
                if (lane == 0) tr[slot] = clock64();
            }
        };
        phase_clock(48, 0.f);
        if (d.flags & F_FIRST) {
            const uint32_t *qw = reinterpret_cast<const uint32_t *>(st.q + r4 * QROW);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                qb[kk][0] = qw[(kk * 16 + c2) / 2];
                qb[kk][1] = qw[(kk * 16 + 8 + c2) / 2];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
            m[0] = m[1] = -INFINITY;
            l[0] = l[1] = 0.f;
        }
        const int base = warp * KP;
        if ((d.flags & F_WRITE) && warp == (d.nrows - 1) / KP) {
            // a2: row lens-1 of this tile is the new token: patch it into the swizzled
            // tile (lanes 0-15 K chunks, 16-31 V chunks) and write it to the cache
            const int rr = d.nrows - 1, ch = lane & 15;
            const uint4 val = reinterpret_cast<const uint4 *>(lane < 16 ? st.knew : st.vnew)[ch];
            *reinterpret_cast<uint4 *>((lane < 16 ? st.k : st.v) + swz(rr, ch, HALF)) = val;
            const size_t dst = (((size_t)d.b * p.Hkv + d.g) * p.max_ctx + d.wrow) * D;
            reinterpret_cast<uint4 *>((lane < 16 ? p.k_w : p.v_w) + dst)[ch] = val;
            __syncwarp();
        }
        if (base < d.nrows) {
            const uint32_t ks_ = smem_u32(st.k), vs_ = smem_u32(st.v);
            const int i4 = lane >> 3, r8 = lane & 7;
            // ---- S^T = K Q^T per 16-key group: A = 16 key rows via ldmatrix (two
            // accumulator chains per group; the NG groups are independent)
            // (branch-free over the groups so their chains interleave; rows past
            // nrows are masked below and their V rows zeroed)
            float x[NG][4];
            bool okg[NG];
            float sa[NG][4], sb[NG][4];
#pragma unroll
            for (int j = 0; j < NG; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) sa[j][i] = sb[j][i] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 8; kk += 2) {
                uint32_t a[NG][4], e[NG][4];
#pragma unroll
                for (int j = 0; j < NG; ++j) {
                    const int key = base + 16 * j + (i4 & 1) * 8 + r8;
                    ldsm_x4(ks_ + swz(key, 2 * kk + (i4 >> 1), HALF), a[j][0], a[j][1], a[j][2], a[j][3]);
                    ldsm_x4(ks_ + swz(key, 2 * kk + 2 + (i4 >> 1), HALF), e[j][0], e[j][1], e[j][2], e[j][3]);
                }
#pragma unroll
                for (int j = 0; j < NG; ++j) {
                    mma16816(sa[j], a[j][0], a[j][1], a[j][2], a[j][3], qb[kk][0], qb[kk][1]);
                    mma16816(sb[j], e[j][0], e[j][1], e[j][2], e[j][3], qb[kk + 1][0], qb[kk + 1][1]);
                }
            }
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                const int gb = base + 16 * j;
                // keys of this thread: gb + r4 (values 0,1) and gb + r4 + 8 (values 2,3)
                const int k0 = gb + r4, k1 = gb + r4 + 8;
                bool ok0 = k0 < d.nrows, ok1 = k1 < d.nrows;
                if (p.mask) {
                    ok0 = ok0 && st.mask[d.moff + (ok0 ? k0 : 0)] != 0;
                    ok1 = ok1 && st.mask[d.moff + (ok1 ? k1 : 0)] != 0;
                }
                x[j][0] = ok0 ? (sa[j][0] + sb[j][0]) * p.scale_log2 : -INFINITY;
                x[j][1] = ok0 ? (sa[j][1] + sb[j][1]) * p.scale_log2 : -INFINITY;
                x[j][2] = ok1 ? (sa[j][2] + sb[j][2]) * p.scale_log2 : -INFINITY;
                x[j][3] = ok1 ? (sa[j][3] + sb[j][3]) * p.scale_log2 : -INFINITY;
                okg[j] = ok0 && ok1;
            }
            // per-head (column) max over the warp's KP keys: lanes with equal lane & 3
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                mx0 = fmaxf(mx0, fmaxf(x[j][0], x[j][2]));
                mx1 = fmaxf(mx1, fmaxf(x[j][1], x[j][3]));
            }
#pragma unroll
            for (int o2 = 4; o2 < 32; o2 <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(FULL_MASK, mx0, o2));
                mx1 = fmaxf(mx1, __shfl_xor_sync(FULL_MASK, mx1, o2));
            }
            phase_clock(49, x[0][0] + x[NG - 1][3]);
            const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);
            const float rf0 = (mn0 == -INFINITY) ? 0.f : mn0, rf1 = (mn1 == -INFINITY) ? 0.f : mn1;
            const float al0 = ex2(m[0] - rf0), al1 = ex2(m[1] - rf1);
            // P.V multiplies bf16(p): sum the same rounded weights
            uint32_t w01[NG], w23[NG];
            float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                const __nv_bfloat162 p01 = __floats2bfloat162_rn(ex2(x[j][0] - rf0), ex2(x[j][1] - rf1));
                const __nv_bfloat162 p23 = __floats2bfloat162_rn(ex2(x[j][2] - rf0), ex2(x[j][3] - rf1));
                ls0 += __low2float(p01) + __low2float(p23);
                ls1 += __high2float(p01) + __high2float(p23);
                w01[j] = *reinterpret_cast<const uint32_t *>(&p01);
                w23[j] = *reinterpret_cast<const uint32_t *>(&p23);
            }
            l[0] = l[0] * al0 + ls0;
            l[1] = l[1] * al1 + ls1;
            m[0] = mn0;
            m[1] = mn1;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                o[i][0] *= al0;
                o[i][1] *= al1;
                o[i][2] *= al0;
                o[i][3] *= al1;
            }
            // masked / out-of-range keys: their V rows may hold anything -> zero them
            bool bad = false;
#pragma unroll
            for (int j = 0; j < NG; ++j) bad = bad || !okg[j];
            if (__any_sync(FULL_MASK, bad)) {
                for (int kr = 0; kr < KP; ++kr) {
                    const int kt = base + kr;
                    bool ok = kt < d.nrows;
                    if (p.mask) ok = ok && st.mask[d.moff + (ok ? kt : 0)] != 0;
                    if (!ok && lane < 16) *reinterpret_cast<uint4 *>(st.v + swz(kt, lane, HALF)) = make_uint4(0, 0, 0, 0);
                }
                __syncwarp();
            }
            // ---- P^T B-fragment: thread needs P[keys c2, c2+1 (+8)][head r4].  The
            // value P[k][n] sits in lane (k & 7) * 4 + n / 2, half n & 1, of p01 (k < 8)
            // or p23 (k >= 8).
            const int srcA = c2 * 4 + (r4 >> 1), srcB = (c2 + 1) * 4 + (r4 >> 1);
            const uint32_t sh = (r4 & 1) ? 16 : 0;
            phase_clock(50, o[7][3] + l[0]);
            uint32_t pb0[NG], pb1[NG];
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                const uint32_t x0 = __shfl_sync(FULL_MASK, w01[j], srcA), x1 = __shfl_sync(FULL_MASK, w01[j], srcB);
                const uint32_t y0 = __shfl_sync(FULL_MASK, w23[j], srcA), y1 = __shfl_sync(FULL_MASK, w23[j], srcB);
                pb0[j] = ((x0 >> sh) & 0xffffu) | (((x1 >> sh) & 0xffffu) << 16);
                pb1[j] = ((y0 >> sh) & 0xffffu) | (((y1 >> sh) & 0xffffu) << 16);
            }
            phase_clock(51, __uint_as_float(pb0[0] ^ pb1[NG - 1]));
            // ---- O^T += V^T P^T: A = V^T (16 dims x 16 keys) via ldmatrix.trans
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a[NG][4];
#pragma unroll
                for (int j = 0; j < NG; ++j) {
                    const int key = base + 16 * j + (i4 >> 1) * 8 + r8;
                    ldsm_x4_t(vs_ + swz(key, 2 * mt + (i4 & 1), HALF), a[j][0], a[j][1], a[j][2], a[j][3]);
                }
#pragma unroll
                for (int j = 0; j < NG; ++j) mma16816(o[mt], a[j][0], a[j][1], a[j][2], a[j][3], pb0[j], pb1[j]);
            }
        }
        __syncwarp();
        phase_clock(52, o[0][0] + o[7][3]);
        if (lane == 0) mbar_arrive(&sm.empty[stage]);
        phase_clock(53, 0.f);
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }

        if (d.flags & F_LAST) {
            // ---- merge the CW warp states in smem (RB = 2: double-buffered, one
            // barrier per item; RB = 1: a second barrier before the buffer is reused).
            // Multi-chunk queries leave an fp32 partial for decode_combine_kernel.
            float ls0 = l[0], ls1 = l[1];
#pragma unroll
            for (int o2 = 4; o2 < 32; o2 <<= 1) {
                ls0 += __shfl_xor_sync(FULL_MASK, ls0, o2);
                ls1 += __shfl_xor_sync(FULL_MASK, ls1, o2);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                sm.red_o[rb][warp][c2][16 * i + r4] = o[i][0];
                sm.red_o[rb][warp][c2 + 1][16 * i + r4] = o[i][1];
                sm.red_o[rb][warp][c2][16 * i + r4 + 8] = o[i][2];
                sm.red_o[rb][warp][c2 + 1][16 * i + r4 + 8] = o[i][3];
            }
            if (lane < 4) {
                sm.red_m[rb][warp][c2] = m[0];
                sm.red_m[rb][warp][c2 + 1] = m[1];
                sm.red_l[rb][warp][c2] = ls0;
                sm.red_l[rb][warp][c2 + 1] = ls1;
            }
            named_bar_sync(1, CW * 32);
          // (head, dims {d0..d0+3} u {d0+64..d0+67}) per thread, CW*32 threads at a
          // time: a half-warp reads 256 contiguous bytes per float4 load
          for (int idx = threadIdx.x; idx < GS * (D / 8); idx += CW * 32) {
            const int hh = idx >> 4, d0 = (idx & 15) * 4;
            float M = -INFINITY;
#pragma unroll
            for (int w2 = 0; w2 < CW; ++w2) M = fmaxf(M, sm.red_m[rb][w2][hh]);
            float Lt = 0.f, Ot[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int w2 = 0; w2 < CW; ++w2) {
                const float mw = sm.red_m[rb][w2][hh];
                const float f = (mw == -INFINITY) ? 0.f : ex2(mw - M);
                Lt = fmaf(f, sm.red_l[rb][w2][hh], Lt);
                const float4 a4 = *reinterpret_cast<const float4 *>(&sm.red_o[rb][w2][hh][d0]);
                const float4 b4 = *reinterpret_cast<const float4 *>(&sm.red_o[rb][w2][hh][d0 + 64]);
                Ot[0] = fmaf(f, a4.x, Ot[0]);
                Ot[1] = fmaf(f, a4.y, Ot[1]);
                Ot[2] = fmaf(f, a4.z, Ot[2]);
                Ot[3] = fmaf(f, a4.w, Ot[3]);
                Ot[4] = fmaf(f, b4.x, Ot[4]);
                Ot[5] = fmaf(f, b4.y, Ot[5]);
                Ot[6] = fmaf(f, b4.z, Ot[6]);
                Ot[7] = fmaf(f, b4.w, Ot[7]);
            }
            const int h = d.g * GS + hh;
            const size_t bh = (size_t)d.b * p.Hq + h;
            if (d.nchunks == 1) {
                const float inv = Lt > 0.f ? 1.f / Lt : 0.f;
                uint2 w0, w1;
                w0.x = pack_bf16(Ot[0] * inv, Ot[1] * inv);
                w0.y = pack_bf16(Ot[2] * inv, Ot[3] * inv);
                w1.x = pack_bf16(Ot[4] * inv, Ot[5] * inv);
                w1.y = pack_bf16(Ot[6] * inv, Ot[7] * inv);
                *reinterpret_cast<uint2 *>(p.out + bh * D + d0) = w0;
                *reinterpret_cast<uint2 *>(p.out + bh * D + d0 + 64) = w1;
            } else {
                float *pp = p.partial + (bh * p.max_chunks + d.c) * (D + PREC_PAD);
                *reinterpret_cast<float4 *>(pp + d0) = make_float4(Ot[0], Ot[1], Ot[2], Ot[3]);
                *reinterpret_cast<float4 *>(pp + d0 + 64) = make_float4(Ot[4], Ot[5], Ot[6], Ot[7]);
                if ((idx & 15) == 0) {
                    pp[D] = M;
                    pp[D + 1] = Lt;
                }
            }
          }
          if constexpr (RB == 1) named_bar_sync(1, CW * 32);   // merge buffer free again
          rb = (rb + 1) % RB;
          if (trace && threadIdx.x == 0 && citem < 8) tr[11 + 4 * citem] = gtimer();
          ++citem;
        }
    }
    if (trace && threadIdx.x == 0) {
        tr[2] = gtimer();
        tr[3] = citem;
    }
}

}  // namespace


template <int CW, int KP, int STAGES, int MINB, int RB = 2>
cudaError_t launch_gqa_v(const DecodeArgs &a, cudaStream_t s) {
    constexpr int TILE = CW * KP, THREADS = (CW + 1) * 32;
    const int num_sms = device_sms();
    const size_t smem = sizeof(Smem<CW, KP, STAGES, RB>) + 1024;
    {
        cudaError_t e = ensure_smem_attr(decode_gqa_kernel<CW, KP, STAGES, RB, MINB>, smem);
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
    p.early = a.early;
    p.trace_slot = g_trace_launch++ % TRACE_L;
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
    // 2-D maps over this layer's cache: [slots*kv_heads*max_ctx rows][128 dims]
    CUtensorMap km, vm;
    const uint64_t dims[2] = {(uint64_t)D, (uint64_t)a.slots * a.kv_heads * a.max_ctx};
    const uint64_t strides[1] = {(uint64_t)D * 2};
    const uint32_t box[2] = {64, TILE};
    if (!encode_bf16_map(&km, a.k, 2, dims, strides, box) || !encode_bf16_map(&vm, a.v, 2, dims, strides, box))
        return cudaErrorInvalidValue;
    cudaError_t e = launch_pdl(decode_gqa_kernel<CW, KP, STAGES, RB, MINB>, dim3(MINB * num_sms), dim3(THREADS), smem, s, km, vm, p);
    if (e != cudaSuccess) return e;
    return launch_gqa_combine(a, s);
}

cudaError_t launch_gqa_experiment(int v, const DecodeArgs &a, cudaStream_t s) {
    switch (v) {
        case 1: return launch_gqa_v<4, 16, 2, 2>(a, s);      // 2 CTAs / SM
        case 5: return launch_gqa_v<4, 16, 5, 1>(a, s);      // deeper ring
        case 6: return launch_gqa_v<4, 32, 2, 1>(a, s);      // 2 MMA chains / warp
        case 9: return launch_gqa_v<8, 16, 2, 1>(a, s);      // 8 consumer warps
        case 10: return launch_gqa_v<4, 32, 3, 1, 1>(a, s);  // 2 chains, 3 stages, 1 merge buffer
        default: return launch_gqa_v<4, 16, 4, 1>(a, s);     // 0: mma.sync, 4 warps x 16 keys
    }
}

}  // namespace baton

// Debug only (not part of include/baton.h): switch the GQA timeline on/off and
// copy it out ([TRACE_L][TRACE_CTAS][TRACE_W] int64, see g_trace).
extern "C" int baton_debug_gqa_trace(int on, void *host, size_t bytes) {
    if (host) {
        if (cudaMemcpyFromSymbol(host, baton::g_trace, bytes < sizeof(baton::g_trace) ? bytes : sizeof(baton::g_trace)) != cudaSuccess)
            return -1;
    }
    if (on >= 0) {
        if (on) {
            static long long zero[baton::TRACE_L][baton::TRACE_CTAS][baton::TRACE_W];
            cudaMemcpyToSymbol(baton::g_trace, zero, sizeof(zero));
        }
        if (cudaMemcpyToSymbol(baton::g_trace_on, &on, sizeof(int)) != cudaSuccess) return -1;
    }
    return 0;
}
