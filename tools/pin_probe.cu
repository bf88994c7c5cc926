// Pinned host allocation cost for one config-5 KKT vector (17.2 GB): cudaMallocHost
// vs mmap + parallel first touch (+ transparent huge pages) + cudaHostRegister.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static void touch(char* p, size_t bytes, int nt) {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([=] {
            const size_t a = bytes / nt * t, b = t == nt - 1 ? bytes : bytes / nt * (t + 1);
            std::memset(p + a, 0, b - a);
        });
    for (auto& x : th) x.join();
}
int main(int argc, char** argv) {
    const size_t bytes = size_t(17) << 30;
    cudaFree(0);
    const int nt = int(std::thread::hardware_concurrency());
    printf("threads %d\n", nt);
    double t = now();
    void* p = nullptr;
    cudaMallocHost(&p, bytes);
    printf("cudaMallocHost %.2f s\n", now() - t);
    t = now();
    std::memset(p, 0, bytes);
    printf("memset 1 thread %.2f s\n", now() - t);
    t = now();
    touch((char*)p, bytes, nt);
    printf("memset %d threads %.2f s\n", nt, now() - t);
    t = now();
    cudaFreeHost(p);
    printf("cudaFreeHost %.2f s\n", now() - t);
    for (int huge = 0; huge < 2; ++huge) {
        t = now();
        char* q = (char*)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (huge) madvise(q, bytes, MADV_HUGEPAGE);
        touch(q, bytes, nt);
        const double t1 = now();
        cudaError_t e = cudaHostRegister(q, bytes, cudaHostRegisterDefault);
        const double t2 = now();
        printf("mmap%s + touch %.2f s + cudaHostRegister %.2f s (%s)\n", huge ? "+THP" : "", t1 - t, t2 - t1,
               cudaGetErrorString(e));
        // H2D bandwidth from it
        void* d = nullptr;
        cudaMalloc(&d, size_t(1) << 30);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int i = 0; i < 8; ++i) cudaMemcpyAsync(d, q + (size_t(i) << 30), size_t(1) << 30, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("  H2D %.1f GB/s\n", 8.0 * 1.073741824 / (ms * 1e-3));
        cudaFree(d);
        t = now();
        cudaHostUnregister(q);
        munmap(q, bytes);
        printf("  unregister+munmap %.2f s\n", now() - t);
    }
    return 0;
}
