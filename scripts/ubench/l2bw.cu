// l2bw.cu -- read bandwidth of L2-resident vs HBM-resident buffers on B200, with the two
// access paths the GS kernel can use: 1-D bulk copies (cp.async.bulk, 16 KB chunks, 4-slot
// mbarrier ring per CTA) and LDG.128.  Each CTA streams a disjoint slice of the buffer
// `reps` times.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kChunk = 16384, kSlots = 4;

__global__ void bulk_read(const char *buf, size_t per_cta, int reps, float *out) {
    extern __shared__ __align__(128) char sm[];
    unsigned long long *bar = reinterpret_cast<unsigned long long *>(sm + kSlots * kChunk);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + i)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const char *base = buf + per_cta * blockIdx.x;
    const int n = (int)(per_cta / kChunk) * reps;
    float acc = 0.f;
    if (threadIdx.x == 0) {
        for (int i = 0; i < n + kSlots; i++) {
            if (i >= kSlots) {  // consume slot of chunk i - kSlots
                const int j = i - kSlots, sl = j % kSlots;
                asm volatile(
                    "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                        su32(bar + sl)),
                    "r"((j / kSlots) & 1));
                acc += reinterpret_cast<float *>(sm + sl * kChunk)[j & 1023];
            }
            if (i < n) {
                const int sl = i % kSlots;
                const char *src = base + (size_t)(i % (per_cta / kChunk)) * kChunk;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + sl)), "r"(kChunk));
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        su32(sm + sl * kChunk)),
                    "l"(src), "r"(kChunk), "r"(su32(bar + sl))
                    : "memory");
            }
        }
        out[blockIdx.x] = acc;
    }
}

__global__ void ldg_read(const float4 *buf, size_t per_cta_f4, int reps, float *out) {
    const float4 *base = buf + per_cta_f4 * blockIdx.x;
    float acc = 0.f;
    for (int r = 0; r < reps; r++)
        for (size_t i = threadIdx.x; i < per_cta_f4; i += blockDim.x * 4) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                size_t k = i + (size_t)u * blockDim.x;
                v[u] = k < per_cta_f4 ? __ldcg(base + k) : make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
    if (acc == 1234.5f) out[blockIdx.x] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t maxb = (size_t)2 << 30;
    char *buf;
    cudaMalloc(&buf, maxb);
    cudaMemset(buf, 0, maxb);
    float *out;
    cudaMalloc(&out, 4096 * 4);
    cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * kChunk + 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t sizes[] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)96 << 20,
                            (size_t)128 << 20, (size_t)1 << 30, (size_t)2 << 30};
    for (int ctas_per_sm : {1, 2, 4}) {
        const int nct = sms * ctas_per_sm;
        for (size_t sz : sizes) {
            size_t per = (sz / nct) / kChunk * kChunk;
            int reps = (int)((8ull << 30) / (per * nct));
            if (reps < 1) reps = 1;
            double bytes = (double)per * nct * reps;
            for (int mode = 0; mode < 2; mode++) {
                for (int w = 0; w < 2; w++) {
                    cudaEventRecord(e0);
                    if (mode == 0)
                        bulk_read<<<nct, 32, kSlots * kChunk + 64>>>(buf, per, reps, out);
                    else
                        ldg_read<<<nct, 256>>>((const float4 *)buf, per / 16, reps, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("ctas/sm=%d size=%7.1f MB mode=%s  %8.1f GB/s\n", ctas_per_sm, sz / 1048576.0,
                       mode ? "ldg " : "bulk", bytes / (ms * 1e-3) / 1e9);
            }
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
