// Throughput / latency probe of legacy mma.sync m16n8k16 bf16 (HMMA.16816) on the
// local GPU: cycles per MMA per SM sub-partition with 1..8 warps per SMSP and 1..8
// independent accumulator chains per warp.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void probe(float *out, long long *cyc, int iters) {
    float c[CHAINS][4];
    for (int j = 0; j < CHAINS; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CHAINS; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    __syncthreads();
    float s = 0.f;
    for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CHAINS>
void run(int warps, float *out, long long *cyc) {
    const int iters = 4096;
    probe<CHAINS><<<1, warps * 32>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double mmas_per_smsp = (double)iters * CHAINS * warps / 4.0;
    printf("{\"warps\": %d, \"chains\": %d, \"cycles\": %lld, \"cycles_per_mma_per_warp\": %.2f, "
           "\"cycles_per_mma_per_smsp\": %.2f}\n",
           warps, CHAINS, h, (double)h / (iters * CHAINS), (double)h / (warps >= 4 ? mmas_per_smsp : iters * CHAINS));
}

int main() {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 1 << 12);
    for (int w : {1, 4, 8, 16, 32}) {
        run<1>(w, out, cyc);
        run<2>(w, out, cyc);
        run<4>(w, out, cyc);
        run<8>(w, out, cyc);
    }
    return 0;
}
