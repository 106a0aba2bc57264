// Micro-benchmark: HBM read bandwidth of cp.async.bulk row streaming (the K1s loading
// pattern) vs plain vectorised loads, over a 164 MB buffer (C3's fp32 input).
// build+run on the box: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk_bw tools/bulk_bw.cu && /tmp/bulk_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_stream(const float* src, size_t n_chunks, int chunk_bytes, int stages, int consume, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint8_t* ring = sm + 128;
    const size_t c0 = n_chunks * blockIdx.x / gridDim.x, c1 = n_chunks * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](size_t c, int s) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(chunk_bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ring + (size_t)s * chunk_bytes)),
                     "l"(reinterpret_cast<const uint8_t*>(src) + c * (size_t)chunk_bytes), "r"(chunk_bytes), "r"(smem_u32(&full[s]))
                     : "memory");
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < stages && c0 + k < c1; ++k) issue(c0 + k, k);
    float acc = 0.f;
    for (size_t c = c0; c < c1; ++c) {
        const size_t k = c - c0;
        const int s = (int)(k % stages);
        const uint32_t par = (uint32_t)((k / stages) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(par) : "memory");
        const float* f = reinterpret_cast<const float*>(ring + (size_t)s * chunk_bytes);
        if (consume)
            for (int i = threadIdx.x; i < chunk_bytes / 4; i += blockDim.x) acc += f[i];
        __syncthreads();
        if (threadIdx.x == 0 && c + stages < c1) issue(c + stages, s);
    }
    if (acc == 123.f) sink[0] = acc;
}

__global__ void plain_stream(const float4* src, size_t n4, float* sink) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(src + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 123.f) sink[0] = acc;
}

int main() {
    const size_t bytes = 10000ull * 4096 * 4;
    float* src;
    float* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(src, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return bytes / (ms / 10 * 1e-3) / 1e9;
    };
    for (int threads : {256, 512})
        for (int mult : {1, 4, 8})
            printf("plain float4 grid-stride: threads %d, %d CTAs/SM: %.0f GB/s\n", threads, mult,
                   timeit([&] { plain_stream<<<sms * mult, threads>>>((const float4*)src, bytes / 16, sink); }));
    for (int chunk : {4096, 16384, 32768, 65536})
        for (int stages : {2, 3, 4, 6})
            for (int per_sm : {1, 2})
                for (int consume : {0, 1}) {
                    size_t smem = 128 + (size_t)stages * chunk;
                    if (smem * per_sm > 227 * 1024) continue;
                    cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    const size_t nch = bytes / chunk;
                    double gbs = timeit([&] { bulk_stream<<<sms * per_sm, 512, smem>>>(src, nch, chunk, stages, consume, sink); });
                    cudaError_t e = cudaGetLastError();
                    printf("bulk chunk %6d stages %d ctas/SM %d consume %d: %.0f GB/s %s\n", chunk, stages, per_sm, consume, gbs,
                           e ? cudaGetErrorString(e) : "");
                }
    return 0;
}
