// host_mem.cu — page-locked host buffers for the host-resident Krylov basis
// (config 5: one KKT vector is 17.2 GB) and fwi_host_alloc.
//
// cudaMallocHost pins page by page: 7.0 s for 17 GB on the B200 boxes, plus
// 1.7 s to free (tools/pin_probe.cu). An anonymous mapping advised onto
// transparent huge pages, faulted in by all host threads and then registered
// with the driver costs 0.27 + 0.38 s (0.33 s to release) and streams H2D at
// the same 55 GB/s.
#include <sys/mman.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace fwi_b200 {

namespace {
std::mutex g_mu;
std::unordered_map<void*, size_t>& registry() {
    static std::unordered_map<void*, size_t> m;
    return m;
}
}  // namespace

void* pinned_alloc(size_t bytes) {
    if (bytes == 0) bytes = 1;
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) throw FwiError(FWI_ERR_OUT_OF_MEMORY, "pinned_alloc: mmap failed");
    madvise(p, bytes, MADV_HUGEPAGE);
    // fault the pages in (zero-filled) from every host thread
    const int nt = bytes >= (size_t(256) << 20) ? std::max(1u, std::min(32u, std::thread::hardware_concurrency())) : 1;
    char* c = static_cast<char*>(p);
    if (nt == 1) {
        std::memset(c, 0, bytes);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([=] {
                const size_t a = bytes / nt * t, b = t == nt - 1 ? bytes : bytes / nt * (t + 1);
                std::memset(c + a, 0, b - a);
            });
        for (auto& x : th) x.join();
    }
    const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        munmap(p, bytes);
        throw FwiError(FWI_ERR_CUDA, std::string("pinned_alloc: cudaHostRegister: ") + cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lk(g_mu);
    registry()[p] = bytes;
    return p;
}

bool pinned_free(void* p) {
    if (!p) return true;
    size_t bytes = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = registry().find(p);
        if (it == registry().end()) return false;
        bytes = it->second;
        registry().erase(it);
    }
    cudaHostUnregister(p);
    munmap(p, bytes);
    return true;
}

}  // namespace fwi_b200
