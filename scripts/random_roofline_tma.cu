// Random-access roofline through the TMA: each warp keeps NB batches of 32 records in flight,
// every record (G bytes at a hashed random offset) fetched by one cp.async.bulk (1-D TMA) into
// shared memory and completed on the batch's mbarrier; compared with plain vector loads
// (scripts/random_roofline.cu).  The question: do bulk copies keep more bytes in flight per SM
// than the load/store unit's outstanding-miss capacity?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rrt scripts/random_roofline_tma.cu && /tmp/rrt 16
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int G, int NB, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_tma_gather(const char* __restrict__ a, uint64_t nrec, int iters, uint32_t* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* buf = sm + (size_t)warp * NB * 32 * G;
    __shared__ __align__(8) uint64_t bars[WARPS][NB];
    if (lane == 0)
        for (int b = 0; b < NB; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp][b])));
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint64_t gw = (blockIdx.x * (uint64_t)WARPS + warp);
    uint32_t acc = 0;
    uint32_t phase[NB];
    for (int b = 0; b < NB; ++b) phase[b] = 0;
    auto issue = [&](int b, int it) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[warp][b])), "r"(32 * G) : "memory");
        __syncwarp();
        const uint64_t r = mix(gw * 1000003ull + it * 32 + lane) & (nrec - 1);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(buf + ((size_t)b * 32 + lane) * G)), "l"(a + r * G), "r"(G), "r"(smem_u32(&bars[warp][b]))
                     : "memory");
    };
    for (int b = 0; b < NB; ++b) issue(b, b);
    for (int it = 0; it < iters; ++it) {
        const int b = it % NB;
        // wait for batch b
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bars[warp][b])), "r"(phase[b]) : "memory");
        phase[b] ^= 1;
        acc ^= *reinterpret_cast<const uint32_t*>(buf + ((size_t)b * 32 + lane) * G);
        __syncwarp();
        if (it + NB < iters) issue(b, it + NB);
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int G, int NB, int WARPS>
double run(const char* a, uint64_t bytes, uint32_t* out) {
    const int iters = 256;
    uint64_t nrec = 1;
    while (nrec * 2 * G <= bytes) nrec *= 2;
    const size_t smem = (size_t)WARPS * NB * 32 * G;
    cudaFuncSetAttribute(k_tma_gather<G, NB, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tma_gather<G, NB, WARPS>, WARPS * 32, smem);
    const int blocks = 148 * (nb > 0 ? nb : 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_tma_gather<G, NB, WARPS><<<blocks, WARPS * 32, smem>>>(a, nrec, iters, out);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(cudaGetLastError())); return 0; }
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_tma_gather<G, NB, WARPS><<<blocks, WARPS * 32, smem>>>(a, nrec, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = (double)blocks * WARPS * 32 * iters * G / (ms / 1e3) / 1e9;
        if (gbs > best) best = gbs;
    }
    printf("  G=%d NB=%d warps/block=%d blocks/SM=%d smem/block=%zu: %.1f GB/s\n", G, NB, WARPS, nb, smem, best);
    return best;
}

int main(int argc, char** argv) {
    const uint64_t bytes = (uint64_t)((argc > 1 ? atof(argv[1]) : 16.0) * (1ull << 30));
    char* a; uint32_t* out;
    if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&out, 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 1, bytes);
    printf("footprint %.2f GiB\n", bytes / 1073741824.0);
    run<64, 4, 8>(a, bytes, out);
    run<64, 8, 8>(a, bytes, out);
    run<64, 16, 4>(a, bytes, out);
    run<128, 8, 4>(a, bytes, out);
    run<32, 16, 8>(a, bytes, out);
    return 0;
}
