// common.cuh -- sm_100a device helpers shared by the libbaton kernels:
// mbarrier + bulk-copy (TMA engine, cp.async.bulk) PTX wrappers and bf16 unpacking.
#pragma once
// Experiment builds (python -m paper_2410_18701_b200.build --experiments) add the
// round-1 sweep variants and the globaltimer debug timelines; the product build
// compiles neither.
#ifndef BATON_EXPERIMENTS
#define BATON_EXPERIMENTS 0
#endif

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdio>

#include <utility>

#define BATON_DEV __device__ __forceinline__

namespace baton {

constexpr unsigned FULL_MASK = 0xffffffffu;

BATON_DEV uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
BATON_DEV void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
BATON_DEV void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
BATON_DEV void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
BATON_DEV void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
BATON_DEV bool mbar_test_wait(uint64_t *bar, uint32_t parity) {   // non-blocking
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
BATON_DEV bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Watchdog: a pipeline deadlock reports the waiting barrier and traps after ~30 s
// (turns a hung GPU into a launch error; long enough for compute-sanitizer racecheck,
// under which a producer can lag its consumers by seconds).  try_wait suspends in hardware,
// so the clock is read only every 1024 unsuccessful tries.
BATON_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    for (uint32_t n = 1;; ++n) {
        if (mbar_try_wait(bar, parity)) return;
        if ((n & 1023) == 0 && clock64() - t0 > 60000000000LL) {
            printf("baton watchdog: block %d thread %d stuck on mbarrier smem+0x%x parity %u\n",
                   blockIdx.x, threadIdx.x, smem_u32(bar), parity);
            __trap();
        }
    }
}

// ---------------------------------------------------------------- bulk copy (TMA engine)
// 1-D bulk copy global -> shared, completion signalled on an mbarrier as tx bytes.
// src, dst 16-B aligned; bytes a multiple of 16.  SASS: UBLKCP.
BATON_DEV void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Same with an L2 eviction-first hint (streamed K/V is read exactly once per layer).
BATON_DEV void bulk_g2s_evict_first(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                    uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
BATON_DEV uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 2^x with the SFU (ex2.approx.ftz): 2^-inf = +0
BATON_DEV float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// gpu-scope acquire-release fetch-add: publishes (cumulatively) everything this
// thread has observed, e.g. partials other threads wrote before an mbarrier it waited on
BATON_DEV void red_add_release_gpu(int32_t *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
BATON_DEV int ld_acquire_gpu(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
BATON_DEV int atom_add_acq_rel_gpu(int32_t *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Programmatic dependent launch: a kernel launched with the PDL attribute may be
// scheduled while its predecessor drains; it must wait before touching anything
// the predecessor writes.  Both are no-ops without the attribute.
BATON_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
BATON_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One lane of a converged warp (elect.sync): uniform-datapath ops under this
// predicate (tcgen05.mma / commit, TMA and bulk copies) issue once, without the per-lane
// ELECT loop ptxas wraps around them under a plain `lane == 0` test
BATON_DEV bool elect_one() {
    uint32_t e;
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(e));
    return e != 0;
}
// named barrier among `nthreads` threads (ids >= 1; 0 is __syncthreads)
BATON_DEV void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- bf16
// two bf16 packed in a uint32 -> two fp32 (exact)
BATON_DEV float bf16lo(uint32_t x) { return __uint_as_float(x << 16); }
BATON_DEV float bf16hi(uint32_t x) { return __uint_as_float(x & 0xffff0000u); }

BATON_DEV uint4 ld_shared_v4(const void *p) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(smem_u32(p)));
    return r;
}

// Launch with programmatic stream serialization (PDL): the kernel may start while
// its predecessor on the stream drains; it calls griddep_wait() before reading
// the predecessor's results.  Also valid inside stream capture (graph edges).
// Per-device launch facts.  Function attributes and SM counts are per device, so
// they are cached per device ordinal (a process may drive several GPUs).
constexpr int kMaxDevices = 64;
inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}
inline int device_sms() {
    static int sms[kMaxDevices] = {};
    const int dev = current_device();
    if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    return sms[dev];
}
// Raise a kernel's dynamic shared memory limit to `bytes` on the current device,
// once per (kernel, device) (no-op at <= 48 KB).  Not a stream operation; the
// launchers call it from their pre-capture dry probes.
inline cudaError_t ensure_smem_attr_raw(const void *kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    struct Entry { const void *k; int dev; int bytes; };
    static Entry tab[256];
    static int n = 0;
    const int dev = current_device();
    for (int i = 0; i < n; ++i)
        if (tab[i].k == kernel && tab[i].dev == dev && tab[i].bytes >= (int)bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess && n < 256) tab[n++] = {kernel, dev, (int)bytes};
    return e;
}
template <typename... KArgs>
cudaError_t ensure_smem_attr(void (*kernel)(KArgs...), size_t bytes) {
    return ensure_smem_attr_raw(reinterpret_cast<const void *>(kernel), bytes);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace baton
