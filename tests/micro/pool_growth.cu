// Diagnostics: cost of growing the stream-ordered pool vs cudaMalloc.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
static double ms(std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}
int main() {
    cudaFree(0);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // (a) one 32 GB async allocation
    auto t = std::chrono::steady_clock::now();
    void *p;
    cudaMallocAsync(&p, 32ull << 30, s);
    cudaStreamSynchronize(s);
    printf("a) mallocAsync 32GB fresh: %.1f ms\n", ms(t));
    t = std::chrono::steady_clock::now();
    cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    printf("   free: %.1f ms\n", ms(t));
    // (b) 500 x 64 MB from the (now reserved) pool
    std::vector<void *> v(500);
    t = std::chrono::steady_clock::now();
    for (auto &q : v) cudaMallocAsync(&q, 64ull << 20, s);
    cudaStreamSynchronize(s);
    printf("b) 500 x 64MB from reserved pool: %.1f ms\n", ms(t));
    for (auto &q : v) cudaFreeAsync(q, s);
    cudaStreamSynchronize(s);
    // (c) 500 x 64 MB beyond the reserve (pool growth in chunks)
    std::vector<void *> w(1000);
    t = std::chrono::steady_clock::now();
    for (auto &q : w) cudaMallocAsync(&q, 64ull << 20, s);
    cudaStreamSynchronize(s);
    printf("c) 1000 x 64MB (32GB reserved, 64GB asked): %.1f ms\n", ms(t));
    for (auto &q : w) cudaFreeAsync(q, s);
    cudaStreamSynchronize(s);
    // (d) plain cudaMalloc 16 GB
    t = std::chrono::steady_clock::now();
    cudaMalloc(&p, 16ull << 30);
    printf("d) cudaMalloc 16GB: %.1f ms\n", ms(t));
    cudaFree(p);
    // (e) many small growths: 20000 x 3 MB
    std::vector<void *> x(20000);
    t = std::chrono::steady_clock::now();
    for (auto &q : x) cudaMallocAsync(&q, 3ull << 20, s);
    cudaStreamSynchronize(s);
    printf("e) 20000 x 3MB: %.1f ms\n", ms(t));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
