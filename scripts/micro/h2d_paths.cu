// H2D upload paths for a freshly written pageable host buffer (the layout arrays' situation):
// pageable cudaMemcpy, cudaHostRegister + cudaMemcpy (+ unregister), and the library's staged copy
// (two 32 MB pinned buffers, multi-threaded memcpy into them).  nvcc -O3 -o h2d_paths h2d_paths.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void fill(char* p, size_t n) {
    std::vector<std::thread> ts;
    for (int t = 0; t < 16; ++t)
        ts.emplace_back([=] { std::memset(p + n * t / 16, t + 1, n / 16); });
    for (auto& t : ts) t.join();
}

int main(int argc, char** argv) {
    const size_t bytes = (argc > 1 ? std::atol(argv[1]) : 600) << 20;
    void* d = nullptr;
    cudaMalloc(&d, bytes);
    cudaFree(nullptr);
    for (int rep = 0; rep < 2; ++rep) {
        {
            char* h = static_cast<char*>(std::malloc(bytes));
            fill(h, bytes);
            const double t0 = now();
            cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
            const double t1 = now();
            std::printf("pageable memcpy: %.1f ms (%.1f GB/s)\n", 1e3 * (t1 - t0), bytes / (t1 - t0) / 1e9);
            std::free(h);
        }
        {
            char* h = static_cast<char*>(std::malloc(bytes));
            fill(h, bytes);
            const double t0 = now();
            cudaHostRegister(h, bytes, cudaHostRegisterDefault);
            const double t1 = now();
            cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
            const double t2 = now();
            cudaHostUnregister(h);
            const double t3 = now();
            std::printf("register %.1f ms + DMA %.1f ms (%.1f GB/s) + unregister %.1f ms = %.1f ms\n", 1e3 * (t1 - t0),
                        1e3 * (t2 - t1), bytes / (t2 - t1) / 1e9, 1e3 * (t3 - t2), 1e3 * (t3 - t0));
            std::free(h);
        }
        {
            char* h = static_cast<char*>(std::malloc(bytes));
            fill(h, bytes);
            constexpr size_t kChunk = 32u << 20;
            void* buf[2];
            cudaEvent_t ev[2];
            for (int i = 0; i < 2; ++i) {
                cudaHostAlloc(&buf[i], kChunk, cudaHostAllocDefault);
                cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
            }
            for (int T : {4, 8, 16}) {
                const double t0 = now();
                int i = 0;
                for (size_t off = 0; off < bytes; off += kChunk, i ^= 1) {
                    const size_t len = std::min(kChunk, bytes - off);
                    cudaEventSynchronize(ev[i]);
                    std::vector<std::thread> ts;
                    for (int t = 0; t < T; ++t)
                        ts.emplace_back([=] {
                            const size_t a = len * t / T, b = len * (t + 1) / T;
                            std::memcpy(static_cast<char*>(buf[i]) + a, h + off + a, b - a);
                        });
                    for (auto& t : ts) t.join();
                    cudaMemcpyAsync(static_cast<char*>(d) + off, buf[i], len, cudaMemcpyHostToDevice, nullptr);
                    cudaEventRecord(ev[i], nullptr);
                }
                cudaDeviceSynchronize();
                const double t1 = now();
                std::printf("staged (%2d threads): %.1f ms (%.1f GB/s)\n", T, 1e3 * (t1 - t0), bytes / (t1 - t0) / 1e9);
            }
            std::free(h);
        }
    }
    return 0;
}
