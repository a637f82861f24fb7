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
//   epilogue: 4 warp states merged in smem; single chunk -> bf16 out, else split-K
//     partials + last-CTA merge (same workspace layout as decode_attention.cu).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "sched.cuh"
#include "tma.h"

namespace baton {

// Debug timeline (off unless baton_debug_gqa_trace(1, ...) was called): per CTA,
// [0] enter [1] work list built [2] exit [3] items [4] smid, then per item k
// [8+4k] item w, [9+4k] first TMA issued, [10+4k] first tile ready, [11+4k] epilogue done.
constexpr int TRACE_CTAS = 1024, TRACE_W = 64;
__device__ int g_trace_on;
__device__ long long g_trace[TRACE_CTAS][TRACE_W];
BATON_DEV long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

namespace {

constexpr int D = 128;
constexpr int GS = 8;                       // q heads per kv head
constexpr int KPW = 16;                     // keys per consumer warp per tile
// CW (consumer warps), STAGES and CTAs/SM are template parameters; a tile has
// TILE = CW * KPW keys and its two 64-dim halves are HALF = TILE * 128 bytes each.
constexpr int F_FIRST = 1, F_LAST = 2, F_END = 4;

struct Desc {
    int32_t b, g, c, nrows, flags, moff, nchunks, wrow;
};

template <int CW>
struct __align__(1024) Stage {
    static constexpr int TILE = CW * KPW;
    static constexpr int HALF = TILE * 128;
    uint8_t k[2 * HALF];
    uint8_t v[2 * HALF];
    __nv_bfloat16 q[GS * D];
    uint8_t mask[TILE + 16];
    Desc desc;
};

template <int CW, int STAGES>
struct Smem {
    Stage<CW> st[STAGES];
    uint64_t full[STAGES], empty[STAGES];
    WorkSched ws;
    alignas(16) float red_o[2][CW][GS][D + 8];     // +8: spread the 8 head rows over the banks
    float red_m[2][CW][GS], red_l[2][CW][GS];
};

struct Params {
    const __nv_bfloat16 *q, *k, *v;
    int32_t *counters;
    const uint8_t *mask;
    const int32_t *lens, *pad;
    __nv_bfloat16 *out;
    float *partial;
    int32_t *tickets;
    int B, Hq, Hkv, max_ctx, max_chunks;
    float scale_log2;
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

template <int CW, int STAGES, int MINB>
__global__ void __launch_bounds__((CW + 1) * 32, MINB)
decode_gqa_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                  const Params p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for the SWIZZLE_128B boxes; offsetting the __shared__ array
    // itself keeps the shared address space visible to the compiler (LDS, not LD)
    constexpr int TILE = CW * KPW, HALF = TILE * 128, THREADS = (CW + 1) * 32;
    Smem<CW, STAGES> &sm =
        *reinterpret_cast<Smem<CW, STAGES> *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool trace = g_trace_on && blockIdx.x < TRACE_CTAS;
    long long *tr = g_trace[trace ? blockIdx.x : 0];
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
    griddep_wait();                 // PDL (see decode_attention.cu)
    griddep_launch_dependents();
    for (int b = blockIdx.x; b < p.B; b += gridDim.x) {
        if (p.lens[b] <= 0) {
            uint4 *o = reinterpret_cast<uint4 *>(p.out + (size_t)b * p.Hq * D);
            for (int i = threadIdx.x; i < p.Hq * D / 8; i += THREADS) o[i] = make_uint4(0, 0, 0, 0);
        }
    }
    __syncthreads();

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
        int w = sched_next(p.counters);
        while (w < total) {
            const int w_next = sched_next(p.counters);   // latency hidden by this item
            int c, g;
            sched_item(sm.ws, w, p.Hkv, b, c, g);
            const int L = sm.ws.lens[b];
            const int nch = (L + CHUNK - 1) / CHUNK;
            const int r0 = c * CHUNK;
            const int rows = min(CHUNK, L - r0);
            const int row_base = (b * p.Hkv + g) * p.max_ctx + r0;   // row in the 2-D tensor map
            const int ntiles = (rows + TILE - 1) / TILE;
            if (trace && titem < (TRACE_W - 8) / 4) {
                tr[8 + 4 * titem] = w;
                tr[9 + 4 * titem] = gtimer();
            }
            ++titem;
            for (int t = 0; t < ntiles; ++t) {
                const int nr = min(TILE, rows - t * TILE);
                mbar_wait(&sm.empty[stage], phase ^ 1);
                Stage<CW> &st = sm.st[stage];
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
                st.desc.b = b;
                st.desc.g = g;
                st.desc.c = c;
                st.desc.nrows = nr;
                st.desc.flags = (t == 0 ? F_FIRST : 0) | (t == ntiles - 1 ? F_LAST : 0);
                st.desc.moff = moff;
                st.desc.nchunks = nch;
                st.desc.wrow = 0;
                mbar_arrive_expect_tx(&sm.full[stage], bytes);
                const int row = row_base + t * TILE;
                tma_load_2d(st.k, &kmap, 0, row, &sm.full[stage]);
                tma_load_2d(st.k + HALF, &kmap, 64, row, &sm.full[stage]);
                tma_load_2d(st.v, &vmap, 0, row, &sm.full[stage]);
                tma_load_2d(st.v + HALF, &vmap, 64, row, &sm.full[stage]);
                if (t == 0)   // the group's 8 query rows (contiguous 2 KB)
                    bulk_g2s(st.q, p.q + ((size_t)b * p.Hq + g * GS) * D, GS * D * 2, &sm.full[stage]);
                if (mbytes) bulk_g2s(st.mask, msrc, mbytes, &sm.full[stage]);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            w = w_next;
        }
        sched_done(p.counters);
        mbar_wait(&sm.empty[stage], phase ^ 1);
        sm.st[stage].desc.flags = F_END;
        mbar_arrive(&sm.full[stage]);
        return;
    }

    // ============================ consumer warps ============================
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
    int citem = 0;
    while (true) {
        mbar_wait(&sm.full[stage], phase);
        Stage<CW> &st = sm.st[stage];
        const Desc d = st.desc;
        if (d.flags & F_END) break;
        if (trace && threadIdx.x == 0 && (d.flags & F_FIRST) && citem < (TRACE_W - 8) / 4)
            tr[10 + 4 * citem] = gtimer();
        if (d.flags & F_FIRST) {
            const uint32_t *qw = reinterpret_cast<const uint32_t *>(st.q + r4 * D);
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
        const int base = warp * KPW;
        if (base < d.nrows) {
            const uint32_t ks_ = smem_u32(st.k), vs_ = smem_u32(st.v);
            const int i4 = lane >> 3, r8 = lane & 7;
            // ---- S^T = K Q^T: A = 16 key rows via ldmatrix (two accumulator chains)
            float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
            {
                const int key = base + (i4 & 1) * 8 + r8;
#pragma unroll
                for (int kk = 0; kk < 8; kk += 2) {
                    uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
                    ldsm_x4(ks_ + swz(key, 2 * kk + (i4 >> 1), HALF), a0, a1, a2, a3);
                    ldsm_x4(ks_ + swz(key, 2 * kk + 2 + (i4 >> 1), HALF), e0, e1, e2, e3);
                    mma16816(sa, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
                    mma16816(sb, e0, e1, e2, e3, qb[kk + 1][0], qb[kk + 1][1]);
                }
            }
            // keys of this thread: r4 (values 0,1) and r4 + 8 (values 2,3)
            const int k0 = base + r4, k1 = base + r4 + 8;
            bool ok0 = k0 < d.nrows, ok1 = k1 < d.nrows;
            if (p.mask) {
                ok0 = ok0 && st.mask[d.moff + (ok0 ? k0 : 0)] != 0;
                ok1 = ok1 && st.mask[d.moff + (ok1 ? k1 : 0)] != 0;
            }
            float x[4];
            x[0] = ok0 ? (sa[0] + sb[0]) * p.scale_log2 : -INFINITY;
            x[1] = ok0 ? (sa[1] + sb[1]) * p.scale_log2 : -INFINITY;
            x[2] = ok1 ? (sa[2] + sb[2]) * p.scale_log2 : -INFINITY;
            x[3] = ok1 ? (sa[3] + sb[3]) * p.scale_log2 : -INFINITY;
            // per-head (column) max over the warp's 16 keys: lanes with equal lane & 3
            float mx0 = fmaxf(x[0], x[2]), mx1 = fmaxf(x[1], x[3]);
#pragma unroll
            for (int o2 = 4; o2 < 32; o2 <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(FULL_MASK, mx0, o2));
                mx1 = fmaxf(mx1, __shfl_xor_sync(FULL_MASK, mx1, o2));
            }
            const float mn0 = fmaxf(m[0], mx0), mn1 = fmaxf(m[1], mx1);
            const float rf0 = (mn0 == -INFINITY) ? 0.f : mn0, rf1 = (mn1 == -INFINITY) ? 0.f : mn1;
            const float al0 = ex2(m[0] - rf0), al1 = ex2(m[1] - rf1);
            // P.V multiplies bf16(p): sum the same rounded weights
            const __nv_bfloat162 p01 = __floats2bfloat162_rn(ex2(x[0] - rf0), ex2(x[1] - rf1));  // key k0
            const __nv_bfloat162 p23 = __floats2bfloat162_rn(ex2(x[2] - rf0), ex2(x[3] - rf1));  // key k1
            l[0] = l[0] * al0 + __low2float(p01) + __low2float(p23);
            l[1] = l[1] * al1 + __high2float(p01) + __high2float(p23);
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
            if (__any_sync(FULL_MASK, !(ok0 && ok1))) {
                for (int kr = 0; kr < KPW; ++kr) {
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
            const uint32_t w01 = *reinterpret_cast<const uint32_t *>(&p01);
            const uint32_t w23 = *reinterpret_cast<const uint32_t *>(&p23);
            const int srcA = c2 * 4 + (r4 >> 1), srcB = (c2 + 1) * 4 + (r4 >> 1);
            const uint32_t sh = (r4 & 1) ? 16 : 0;
            const uint32_t x0 = __shfl_sync(FULL_MASK, w01, srcA), x1 = __shfl_sync(FULL_MASK, w01, srcB);
            const uint32_t y0 = __shfl_sync(FULL_MASK, w23, srcA), y1 = __shfl_sync(FULL_MASK, w23, srcB);
            const uint32_t pb0 = ((x0 >> sh) & 0xffffu) | (((x1 >> sh) & 0xffffu) << 16);
            const uint32_t pb1 = ((y0 >> sh) & 0xffffu) | (((y1 >> sh) & 0xffffu) << 16);
            // ---- O^T += V^T P^T: A = V^T (16 dims x 16 keys) via ldmatrix.trans
            {
                const int key = base + (i4 >> 1) * 8 + r8;
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_t(vs_ + swz(key, 2 * mt + (i4 & 1), HALF), a0, a1, a2, a3);
                    mma16816(o[mt], a0, a1, a2, a3, pb0, pb1);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[stage]);
        if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
        }

        if (d.flags & F_LAST) {
            // ---- merge the 4 warp states (double-buffered smem: one barrier per item).
            // Multi-chunk queries leave an fp32 partial; decode_combine_kernel (next in
            // the stream, PDL) merges chunks in order -- no tickets, no waiting here.
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
          // (head, 8-dim block) pairs, CW*32 threads at a time
          for (int idx = threadIdx.x; idx < GS * (D / 8); idx += CW * 32) {
            const int hh = idx >> 4, d0 = (idx & 15) * 8;
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
                const float4 b4 = *reinterpret_cast<const float4 *>(&sm.red_o[rb][w2][hh][d0 + 4]);
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
                uint4 w4;
                w4.x = pack_bf16(Ot[0] * inv, Ot[1] * inv);
                w4.y = pack_bf16(Ot[2] * inv, Ot[3] * inv);
                w4.z = pack_bf16(Ot[4] * inv, Ot[5] * inv);
                w4.w = pack_bf16(Ot[6] * inv, Ot[7] * inv);
                *reinterpret_cast<uint4 *>(p.out + bh * D + d0) = w4;
            } else {
                float *pp = p.partial + (bh * p.max_chunks + d.c) * (D + PREC_PAD);
                *reinterpret_cast<float4 *>(pp + d0) = make_float4(Ot[0], Ot[1], Ot[2], Ot[3]);
                *reinterpret_cast<float4 *>(pp + d0 + 4) = make_float4(Ot[4], Ot[5], Ot[6], Ot[7]);
                if ((idx & 15) == 0) {
                    pp[D] = M;
                    pp[D + 1] = Lt;
                }
            }
          }
          rb ^= 1;
          if (trace && threadIdx.x == 0 && citem < (TRACE_W - 8) / 4) tr[11 + 4 * citem] = gtimer();
          ++citem;
        }
    }
    if (trace && threadIdx.x == 0) {
        tr[2] = gtimer();
        tr[3] = citem;
    }
}

// Split-K merge for multi-chunk queries: one warp per (slot, q head), chunks merged
// in ascending order (batch-invariant).  Single-chunk queries were written directly.
__global__ void __launch_bounds__(128) decode_combine_kernel(const int32_t *__restrict__ lens,
                                                             const float *__restrict__ partial,
                                                             __nv_bfloat16 *__restrict__ out, int B,
                                                             int Hq, int max_chunks) {
    griddep_wait();
    griddep_launch_dependents();
    const int pair = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (pair >= B * Hq) return;
    const int b = pair / Hq;
    const int L = lens[b];
    const int nch = (L + CHUNK - 1) / CHUNK;
    if (nch <= 1) return;
    const float *pp = partial + (size_t)pair * max_chunks * (D + PREC_PAD);
    float Mc = -INFINITY;
    for (int c = 0; c < nch; ++c) Mc = fmaxf(Mc, pp[c * (D + PREC_PAD) + D]);
    float Lc = 0.f;
    float4 Oc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = 0; c < nch; ++c) {
        const float mc = pp[c * (D + PREC_PAD) + D];
        const float f = (mc == -INFINITY) ? 0.f : ex2(mc - Mc);
        Lc = fmaf(f, pp[c * (D + PREC_PAD) + D + 1], Lc);
        const float4 v = *reinterpret_cast<const float4 *>(pp + c * (D + PREC_PAD) + lane * 4);
        Oc.x = fmaf(f, v.x, Oc.x);
        Oc.y = fmaf(f, v.y, Oc.y);
        Oc.z = fmaf(f, v.z, Oc.z);
        Oc.w = fmaf(f, v.w, Oc.w);
    }
    const float inv = Lc > 0.f ? 1.f / Lc : 0.f;
    uint2 w;
    w.x = pack_bf16(Oc.x * inv, Oc.y * inv);
    w.y = pack_bf16(Oc.z * inv, Oc.w * inv);
    *reinterpret_cast<uint2 *>(out + (size_t)pair * D + lane * 4) = w;
}

}  // namespace

bool gqa_supported(int q_heads, int kv_heads, int head_dim) {
    return head_dim == D && kv_heads > 0 && q_heads == GS * kv_heads;
}

template <int CW, int STAGES, int MINB>
cudaError_t launch_gqa_v(const DecodeArgs &a, cudaStream_t s) {
    constexpr int TILE = CW * KPW, THREADS = (CW + 1) * 32;
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const size_t smem = sizeof(Smem<CW, STAGES>) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(decode_gqa_kernel<CW, STAGES, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (a.dry) return cudaSuccess;
    Params p;
    p.q = static_cast<const __nv_bfloat16 *>(a.q);
    p.k = static_cast<const __nv_bfloat16 *>(a.k);
    p.v = static_cast<const __nv_bfloat16 *>(a.v);
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
    if (a.k_new) {   // a2 as its own (PDL-chained) launch before the attention
        cudaError_t e = launch_append_kv(const_cast<void *>(a.k), const_cast<void *>(a.v), a.k_new, a.v_new,
                                         a.lens, a.slots, a.kv_heads, a.head_dim, a.max_ctx, s);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = launch_pdl(decode_gqa_kernel<CW, STAGES, MINB>, dim3(MINB * num_sms), dim3(THREADS), smem, s, km, vm, p);
    if (e != cudaSuccess) return e;
    const int pairs = a.slots * a.q_heads;
    return launch_pdl(decode_combine_kernel, dim3((pairs + 3) / 4), dim3(128), 0, s, a.lens,
                      (const float *)a.partial, static_cast<__nv_bfloat16 *>(a.out), a.slots,
                      a.q_heads, a.max_chunks);
}

cudaError_t launch_decode_gqa(const DecodeArgs &a, cudaStream_t s) {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("BATON_GQA_VARIANT");
        v = e ? atoi(e) : 0;
    }
    switch (v) {
        case 1: return launch_gqa_v<4, 2, 2>(a, s);
        case 2: return launch_gqa_v<2, 2, 3>(a, s);
        case 3: return launch_gqa_v<2, 3, 2>(a, s);
        case 4: return launch_gqa_v<1, 4, 4>(a, s);
        case 5: return launch_gqa_v<4, 5, 1>(a, s);
        default: return launch_gqa_v<4, 4, 1>(a, s);
    }
}

}  // namespace baton

// Debug only (not part of include/baton.h): switch the GQA timeline on/off and
// copy it out ([TRACE_CTAS][TRACE_W] int64, see g_trace).
extern "C" int baton_debug_gqa_trace(int on, void *host, size_t bytes) {
    if (host) {
        if (cudaMemcpyFromSymbol(host, baton::g_trace, bytes < sizeof(baton::g_trace) ? bytes : sizeof(baton::g_trace)) != cudaSuccess)
            return -1;
    }
    if (on >= 0) {
        if (on) {
            static long long zero[baton::TRACE_CTAS][baton::TRACE_W];
            cudaMemcpyToSymbol(baton::g_trace, zero, sizeof(zero));
        }
        if (cudaMemcpyToSymbol(baton::g_trace_on, &on, sizeof(int)) != cudaSuccess) return -1;
    }
    return 0;
}
