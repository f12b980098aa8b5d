// DRAM bytes moved per random access of G bytes (G = 4 .. 128) on this GPU: every thread
// reads independent G-byte items at hashed random offsets of a 16 GiB buffer (far larger than
// L2), ILP items in flight.  Run under
//   ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:k_rand
// and divide dram__bytes_read.sum by the printed access count: the DRAM cost of one random
// 4 / 8 B read (the MDRW slot word, its metadata and col entry) vs the 32 B sector it asks for.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rg scripts/random_granule.cu && /tmp/rg
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}

// 4 B loads with a chosen cache operator (F): 0 __ldg (ld.global.nc), 1 ld.global.ca,
// 2 ld.global.cg (L2 only), 3 ld.global.cs (evict first), 4 ld.global.nc.L1::no_allocate,
// 5 ld.global.nc.L2::64B, 6 ld.global.nc.L2::128B
template <int F>
__device__ __forceinline__ uint32_t ld4(const uint32_t* p) {
    uint32_t v;
    if constexpr (F == 0) v = __ldg(p);
    else if constexpr (F == 1) asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (F == 2) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (F == 3) asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (F == 4) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if constexpr (F == 5) asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else asm volatile("ld.global.nc.L2::128B.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <int F>
__global__ void k_rand4(const unsigned char* __restrict__ a, uint64_t nitem, int iters, uint32_t* out) {
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    uint32_t acc = 0;
    constexpr int ILP = 8;
    for (int it = 0; it < iters; it += ILP) {
        uint32_t v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            const uint64_t r = mix(tid * 1000003ull + it + k) & (nitem - 1);
            v[k] = ld4<F>(reinterpret_cast<const uint32_t*>(a + r * 4));
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc ^= v[k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int G>
__global__ void k_rand(const unsigned char* __restrict__ a, uint64_t nitem, int iters, uint32_t* out) {
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    uint32_t acc = 0;
    constexpr int ILP = 8;
    for (int it = 0; it < iters; it += ILP) {
        uint32_t v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            const uint64_t r = mix(tid * 1000003ull + it + k) & (nitem - 1);
            const unsigned char* p = a + r * G;
            if constexpr (G == 4) v[k] = __ldg(reinterpret_cast<const uint32_t*>(p));
            else if constexpr (G == 8) { const uint2 q = __ldg(reinterpret_cast<const uint2*>(p)); v[k] = q.x ^ q.y; }
            else {
                uint32_t x = 0;
#pragma unroll
                for (int j = 0; j < G / 16; ++j) { const uint4 q = __ldg(reinterpret_cast<const uint4*>(p) + j); x ^= q.x ^ q.w; }
                v[k] = x;
            }
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc ^= v[k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int G>
void run(const unsigned char* a, uint64_t bytes, uint32_t* out) {
    const int threads = 256, blocks = 148 * 8, iters = 64;
    uint64_t nitem = 1;
    while (nitem * 2 * G <= bytes) nitem *= 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rand<G><<<blocks, threads>>>(a, nitem, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double acc = static_cast<double>(blocks) * threads * iters;
    printf("G=%3d B accesses=%.0f ms=%.3f Gaccess/s=%.2f requested GB/s=%.1f\n", G, acc, ms, acc / ms / 1e6,
           acc * G / ms / 1e6);
}

template <int F>
void run4(const unsigned char* a, uint64_t bytes, uint32_t* out) {
    const int threads = 256, blocks = 148 * 8, iters = 64;
    const uint64_t nitem = bytes / 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rand4<F><<<blocks, threads>>>(a, nitem, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double acc = static_cast<double>(blocks) * threads * iters;
    printf("4 B flavour %d footprint %.0f MiB: Gaccess/s=%.2f\n", F, bytes / 1048576.0, acc / ms / 1e6);
}

int main() {
    const uint64_t bytes = 16ull << 30;
    unsigned char* a = nullptr;
    uint32_t* out = nullptr;
    if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&out, 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 1, bytes);
    run<4>(a, bytes, out);
    run<8>(a, bytes, out);
    run<16>(a, bytes, out);
    run<32>(a, bytes, out);
    run<64>(a, bytes, out);
    run<128>(a, bytes, out);
    const uint64_t fbs[2] = {bytes, 1ull << 30};   // 16 GiB and 1 GiB footprints (TLB reach)
    for (uint64_t fb : fbs) {
        run4<0>(a, fb, out); run4<1>(a, fb, out); run4<2>(a, fb, out); run4<3>(a, fb, out);
        run4<4>(a, fb, out); run4<5>(a, fb, out); run4<6>(a, fb, out);
    }
    cudaDeviceSynchronize();
    return 0;
}
