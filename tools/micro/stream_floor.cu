// Calibration: how long do simple 1M-element passes take on this B200 (event-timed,
// back to back)?  copy of B bytes, and 1M returning atomicAdds into 1M random bins.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/stream_floor.cu -o tools/micro/stream_floor
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_hist(const uint32_t* __restrict__ key, uint32_t* cnt, uint32_t* rank, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rank[i] = atomicAdd(cnt + key[i], 1u);
}
__global__ void k_touch(const uint32_t* __restrict__ a, uint32_t* __restrict__ b, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i] + 1;
}
__global__ void k_empty() {}

int main()
{
    const int N = 1 << 20;
    size_t big = 64ull << 20;
    int4 *a, *b;
    cudaMalloc(&a, big); cudaMalloc(&b, big);
    uint32_t *key, *cnt, *rank, *u, *v;
    cudaMalloc(&key, 4 * N); cudaMalloc(&cnt, 4 * N); cudaMalloc(&rank, 4 * N);
    cudaMalloc(&u, 4 * N); cudaMalloc(&v, 4 * N);
    std::vector<uint32_t> h(N);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < N; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (uint32_t)(x % N); }
    cudaMemcpy(key, h.data(), 4 * N, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto t = [&](auto f, const char* name) {
        f(); cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 20; r++) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %8.2f us\n", name, ms * 1000 / 20);
    };
    t([&] { k_empty<<<1, 32>>>(); }, "empty launch");
    for (size_t mb : {4, 8, 16, 32, 64}) {
        size_t n4 = (mb << 20) / 16;
        char nm[64]; snprintf(nm, 64, "copy %zu MB (read %zu + write %zu)", mb, mb, mb);
        t([&] { k_copy<<<148 * 8, 256>>>(a, b, n4); }, nm);
    }
    t([&] { k_touch<<<N / 256, 256>>>(u, v, N); }, "1M x 4B read+write (1 per thread)");
    t([&] { cudaMemsetAsync(cnt, 0, 4 * N); k_hist<<<N / 256, 256>>>(key, cnt, rank, N); }, "memset + 1M returning atomicAdd");
    return 0;
}
