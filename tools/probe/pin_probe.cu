// pin_probe.cu -- how fast can the host store be pinned?  cudaHostAlloc vs
// mmap + transparent huge pages + parallel first touch + cudaHostRegister,
// and the H2D / D2H bandwidth from each (the out-of-core roofline).
//   nvcc -O2 -o /tmp/pin_probe tools/probe/pin_probe.cu -lpthread && /tmp/pin_probe 16
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void touch(char* p, size_t n, int nt)
{
    std::vector<std::thread> th;
    for (int t = 0; t < nt; t++)
        th.emplace_back([=] {
            const size_t a = n / nt * t, b = t == nt - 1 ? n : n / nt * (t + 1);
            for (size_t i = a; i < b; i += 4096) p[i] = 0;
        });
    for (auto& x : th) x.join();
}

static void bw(const char* tag, char* h, size_t n)
{
    const size_t chunk = std::min<size_t>(n, (size_t)2 << 30);
    void* d;
    cudaMalloc(&d, chunk);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best_h2d = 0, best_d2h = 0;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, chunk, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best_h2d = std::max(best_h2d, (float)(chunk / (ms / 1e3) / 1e9));
        cudaEventRecord(a);
        cudaMemcpyAsync(h + (n - chunk), d, chunk, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        best_d2h = std::max(best_d2h, (float)(chunk / (ms / 1e3) / 1e9));
    }
    printf("%s: H2D %.1f GB/s, D2H %.1f GB/s\n", tag, best_h2d, best_d2h);
    cudaFree(d);
}

int main(int argc, char** argv)
{
    const size_t gb = argc > 1 ? atol(argv[1]) : 16;
    const size_t n = gb << 30;
    const int nt = (int)std::thread::hardware_concurrency();
    cudaFree(0);
    {
        double t0 = now();
        void* p;
        cudaError_t e = cudaHostAlloc(&p, n, cudaHostAllocDefault);
        double t1 = now();
        printf("cudaHostAlloc %zu GiB: %.2f s (%s)\n", gb, t1 - t0, cudaGetErrorString(e));
        if (e == cudaSuccess) {
            bw("cudaHostAlloc", (char*)p, n);
            t0 = now();
            cudaFreeHost(p);
            printf("cudaFreeHost: %.2f s\n", now() - t0);
        }
    }
    for (int huge = 0; huge < 2; huge++) {
        double t0 = now();
        char* p = (char*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (huge) madvise(p, n, MADV_HUGEPAGE);
        touch(p, n, nt);
        double t1 = now();
        cudaError_t e = cudaHostRegister(p, n, cudaHostRegisterDefault);
        double t2 = now();
        printf("mmap%s + touch(%d threads) %.2f s + cudaHostRegister %.2f s = %.2f s (%s)\n", huge ? "+THP" : "", nt,
               t1 - t0, t2 - t1, t2 - t0, cudaGetErrorString(e));
        if (e == cudaSuccess) {
            bw(huge ? "registered THP" : "registered 4K", p, n);
            t0 = now();
            cudaHostUnregister(p);
            printf("cudaHostUnregister: %.2f s\n", now() - t0);
        }
        munmap(p, n);
    }
    return 0;
}
