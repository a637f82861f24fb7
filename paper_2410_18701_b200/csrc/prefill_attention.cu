// prefill_attention.cu -- a8: causal attention of a newly inserted query over its
// own prompt, the "prefilling" that Baton decouples from decoding ("all
// original queries awaiting processing are initially prefilled by the model";
// P:L215 asynchronous P&D decoupling).  Row i of the output is the textbook
// SDPA of query token i over keys 0..i -- the decode attention of every
// prefix at once, a dense contraction, so it runs on the 5th-gen tensor cores.
//
// One CTA per (q head, 128-query tile).  Warp roles:
//   warp 4   TMA producer: Q tile once, then K/V tiles of 128 keys into a 2-stage
//            ring (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier tx-counts)
//   warp 5   MMA issuer (one elected thread): S = Q K^T (M=128,N=128,K=16 x8)
//            into TMEM, then O += P V (M=128,N=128,K=16 x8) into TMEM, each
//            completion published with tcgen05.commit -> mbarrier
//   warps 0-3 softmax: thread = query row; tcgen05.ld of its S row, causal mask,
//            online max/sum (exp2), P -> bf16 into the K-major SW128 smem layout
//            the next MMA reads, O rescale in TMEM (tcgen05.ld/st), epilogue.
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace baton {
namespace {

constexpr int PF_M = 128;         // queries per tile (UMMA M, TMEM lanes)
constexpr int PF_N = 128;         // keys per tile (UMMA N of S, K of PV)
constexpr int PF_D = 128;         // head_dim
constexpr int PF_THREADS = 192;   // 4 softmax warps + producer warp + MMA warp
constexpr int TILE_BYTES = PF_M * PF_D * 2;     // 32 KB (two 16 KB swizzle regions)
constexpr int REGION = TILE_BYTES / 2;           // 16 KB: 128 rows x 64 bf16

struct __align__(1024) PfSmem {
    uint8_t q[TILE_BYTES];
    uint8_t k[2][TILE_BYTES];
    uint8_t v[2][TILE_BYTES];
    uint8_t p[TILE_BYTES];
    uint64_t bar_q, kv_full[2], kv_empty[2], s_full, s_free, p_full, o_done;
    uint32_t tmem_base;
};

// ------------------------------------------------------------------ tcgen05 / TMA PTX
BATON_DEV void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
BATON_DEV void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
BATON_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
BATON_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
BATON_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

BATON_DEV void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
BATON_DEV void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 columns of 32-bit: thread t of the warp gets row (lane base + t), 32 columns
BATON_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
BATON_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
BATON_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
BATON_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor (tcgen05 "smem descriptor"): start >> 4 in
// [0,14), LBO >> 4 in [16,30), SBO >> 4 in [32,46), version 1 in [46,48),
// layout type in [61,64) (2 = 128-byte swizzle).
BATON_DEV uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// Instruction descriptor, kind::f16: D fp32, A/B bf16, K- or MN-major B.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct PfParams {
    int Hq, Hkv, len, n_mtiles;
    float scale_log2;
    __nv_bfloat16 *out;
};

__global__ void __launch_bounds__(PF_THREADS, 1)
prefill_attention_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const PfParams p) {
    extern __shared__ uint8_t smem_raw[];
    PfSmem &sm = *reinterpret_cast<PfSmem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // heavy tiles (near the diagonal end) first
    const int mt = p.n_mtiles - 1 - (int)(blockIdx.x % p.n_mtiles);
    const int h = blockIdx.x / p.n_mtiles;
    const int g = h * p.Hkv / p.Hq;
    const int q0 = mt * PF_M;
    const int n_kt = (min(q0 + PF_M, p.len) + PF_N - 1) / PF_N;   // key tiles up to the diagonal

    if (threadIdx.x == 0) {
        mbar_init(&sm.bar_q, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.kv_full[s], 1);
            mbar_init(&sm.kv_empty[s], 1);
        }
        mbar_init(&sm.s_full, 1);
        mbar_init(&sm.s_free, 128);
        mbar_init(&sm.p_full, 128);
        mbar_init(&sm.o_done, 1);
        fence_mbar_init();
    }
    if (warp == 0) {   // TMEM: S in columns [0,128), O in [128,256)
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
        if (lane == 0) {
            prefetch_tmap(&tm_q);
            prefetch_tmap(&tm_k);
            prefetch_tmap(&tm_v);
            mbar_arrive_expect_tx(&sm.bar_q, TILE_BYTES);
            tma_load_3d(sm.q, &tm_q, 0, q0, h, &sm.bar_q);
            tma_load_3d(sm.q + REGION, &tm_q, 64, q0, h, &sm.bar_q);
            for (int j = 0; j < n_kt; ++j) {
                const int s = j & 1;
                if (j >= 2) mbar_wait(&sm.kv_empty[s], ((j >> 1) + 1) & 1);
                mbar_arrive_expect_tx(&sm.kv_full[s], 2 * TILE_BYTES);
                tma_load_3d(sm.k[s], &tm_k, 0, j * PF_N, g, &sm.kv_full[s]);
                tma_load_3d(sm.k[s] + REGION, &tm_k, 64, j * PF_N, g, &sm.kv_full[s]);
                tma_load_3d(sm.v[s], &tm_v, 0, j * PF_N, g, &sm.kv_full[s]);
                tma_load_3d(sm.v[s] + REGION, &tm_v, 64, j * PF_N, g, &sm.kv_full[s]);
            }
        }
    } else if (warp == 5) {
        // ======================= MMA issuer =======================
        if (lane == 0) {
            constexpr uint32_t idS = idesc_bf16(PF_M, PF_N, 0);   // B = K tile, K-major
            constexpr uint32_t idO = idesc_bf16(PF_M, PF_D, 1);   // B = V tile, MN-major
            const uint32_t qa = smem_u32(sm.q), pa = smem_u32(sm.p);
            mbar_wait(&sm.bar_q, 0);
            for (int j = 0; j < n_kt; ++j) {
                const int s = j & 1;
                mbar_wait(&sm.kv_full[s], (j >> 1) & 1);
                if (j > 0) mbar_wait(&sm.s_free, (j - 1) & 1);   // softmax has read S_{j-1}
                tc_fence_after();
                const uint32_t ka = smem_u32(sm.k[s]), va = smem_u32(sm.v[s]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {   // K = head_dim in steps of 16 (32 B)
                    const uint32_t off = (k >> 2) * REGION + (k & 3) * 32;
                    umma_f16(tS, smem_desc(qa + off, 16, 1024), smem_desc(ka + off, 16, 1024), idS, k > 0);
                }
                umma_commit(&sm.s_full);
                mbar_wait(&sm.p_full, j & 1);                   // P_j written, O rescaled
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < 8; ++k) {   // K = keys in steps of 16
                    const uint32_t aoff = (k >> 2) * REGION + (k & 3) * 32;
                    umma_f16(tO, smem_desc(pa + aoff, 16, 1024),
                             smem_desc(va + k * 2048, REGION, 1024), idO, (j > 0 || k > 0));
                }
                umma_commit(&sm.o_done);
                umma_commit(&sm.kv_empty[s]);
            }
        }
    } else {
        // ======================= softmax warps 0-3 =======================
        const int row = warp * 32 + lane;            // query row within the tile = TMEM lane
        const int qi = q0 + row;
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        float m = -INFINITY, l = 0.f;
        uint32_t pk[64];                              // P row packed bf16x2
        for (int j = 0; j < n_kt; ++j) {
            mbar_wait(&sm.s_full, j & 1);
            tc_fence_after();
            const int kbase = j * PF_N;
            const bool diag = kbase + PF_N > q0;      // tile touches the causal diagonal
            // pass 1: row max
            float mx = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32];
                tmem_ld32(tS + lane_off + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int kj = kbase + c * 32 + i;
                    float x = __uint_as_float(r[i]) * p.scale_log2;
                    if (diag && kj > qi) x = -INFINITY;
                    mx = fmaxf(mx, x);
                }
            }
            const float m_new = fmaxf(m, mx);
            const float alpha = ex2(m - m_new);
            // pass 2: probabilities
            float rs = 0.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32];
                tmem_ld32(tS + lane_off + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    const int kj = kbase + c * 32 + i;
                    float x0 = __uint_as_float(r[i]) * p.scale_log2;
                    float x1 = __uint_as_float(r[i + 1]) * p.scale_log2;
                    if (diag && kj > qi) x0 = -INFINITY;
                    if (diag && kj + 1 > qi) x1 = -INFINITY;
                    const float e0 = ex2(x0 - m_new), e1 = ex2(x1 - m_new);
                    const __nv_bfloat162 b = __floats2bfloat162_rn(e0, e1);
                    // the PV MMA consumes bf16 P: accumulate the sum of what it multiplies
                    rs += __low2float(b) + __high2float(b);
                    pk[c * 16 + i / 2] = *reinterpret_cast<const uint32_t *>(&b);
                }
            }
            l = l * alpha + rs;
            m = m_new;
            tc_fence_before();
            mbar_arrive(&sm.s_free);
            if (j > 0) {
                mbar_wait(&sm.o_done, (j - 1) & 1);   // PV_{j-1} done: O stable, P buffer free
                tc_fence_after();
                // warp-uniform: tcgen05.ld/st are .sync.aligned (all 32 lanes converged)
                if (__any_sync(FULL_MASK, alpha != 1.f)) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t r[32];
                        tmem_ld32(tO + lane_off + c * 32, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                        tmem_st32(tO + lane_off + c * 32, r);
                    }
                    tmem_wait_st();
                }
            }
            // P row -> smem, K-major SWIZZLE_128B: keys [64a, 64a+64) in region a,
            // 16-B chunk c of row r at chunk position c ^ (r & 7)
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const int region = c >> 3, chunk = c & 7;
                uint8_t *dst = sm.p + region * REGION + row * 128 + ((chunk ^ (row & 7)) << 4);
                *reinterpret_cast<uint4 *>(dst) =
                    make_uint4(pk[c * 4], pk[c * 4 + 1], pk[c * 4 + 2], pk[c * 4 + 3]);
            }
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(&sm.p_full);
        }
        // epilogue: O / l -> bf16
        mbar_wait(&sm.o_done, (n_kt - 1) & 1);
        tc_fence_after();
        const float inv = 1.f / l;
        __nv_bfloat16 *orow = p.out + ((size_t)h * p.len + qi) * PF_D;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(tO + lane_off + c * 32, r);
            tmem_wait_ld();
            if (qi < p.len) {
                uint32_t w[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(r[2 * i]) * inv,
                                                                   __uint_as_float(r[2 * i + 1]) * inv);
                    w[i] = *reinterpret_cast<const uint32_t *>(&b);
                }
                uint4 *o4 = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                for (int i = 0; i < 4; ++i) o4[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}


PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

bool make_map(CUtensorMap *m, const void *base, int heads, int len) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)PF_D, (cuuint64_t)len, (cuuint64_t)heads};
    cuuint64_t strides[2] = {(cuuint64_t)PF_D * 2, (cuuint64_t)len * PF_D * 2};
    cuuint32_t box[3] = {64, 128, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

bool prefill_supported(int head_dim) { return head_dim == PF_D; }

cudaError_t launch_prefill_attention(const void *q, const void *k, const void *v, void *out, int len,
                                     int q_heads, int kv_heads, int head_dim, float scale,
                                     cudaStream_t s) {
    if (head_dim != PF_D || len < 1) return cudaErrorInvalidValue;
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, q, q_heads, len) || !make_map(&mk, k, kv_heads, len) || !make_map(&mv, v, kv_heads, len))
        return cudaErrorInvalidValue;
    PfParams p;
    p.Hq = q_heads;
    p.Hkv = kv_heads;
    p.len = len;
    p.n_mtiles = (len + PF_M - 1) / PF_M;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.out = static_cast<__nv_bfloat16 *>(out);
    const size_t smem = sizeof(PfSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(prefill_attention_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    prefill_attention_kernel<<<p.n_mtiles * q_heads, PF_THREADS, smem, s>>>(mq, mk, mv, p);
    return cudaGetLastError();
}

}  // namespace baton
