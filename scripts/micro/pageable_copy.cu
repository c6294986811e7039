// Micro-benchmark (development): D2H of a 256^3 FP32 level (device pitch 256 floats) into a
// pageable, halo-padded host block (the drop-in's Field layout, halo 4), three ways:
//   pitched : one cudaMemcpy3D into pageable memory (the driver stages it)
//   register: cudaHostRegister the host block, cudaMemcpy3D at pinned speed, unregister
//   staged  : packed chunks into a pinned double buffer + multi-threaded host scatter
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o pageable_copy pageable_copy.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));     \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    const int n = 256, halo = 4, np = n + 2 * halo;
    const size_t lvl = size_t(n) * n * n;
    float* d = nullptr;
    CK(cudaMalloc(&d, lvl * 4));
    CK(cudaMemset(d, 1, lvl * 4));
    std::vector<float> host(size_t(np) * np * np, 0.f);  // pageable, touched
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    auto pitched = [&]() -> int {
        cudaMemcpy3DParms cp{};
        cp.srcPtr = make_cudaPitchedPtr(d, 4 * n, 4 * n, n);
        cp.dstPtr = make_cudaPitchedPtr(host.data(), 4 * np, 4 * np, np);
        cp.dstPos = make_cudaPos(4 * halo, halo, halo);
        cp.extent = make_cudaExtent(4 * n, n, n);
        cp.kind = cudaMemcpyDeviceToHost;
        CK(cudaMemcpy3DAsync(&cp, s));
        CK(cudaStreamSynchronize(s));
        return 0;
    };
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = now();
        if (pitched()) return 1;
        double t1 = now();
        CK(cudaHostRegister(host.data(), host.size() * 4, cudaHostRegisterDefault));
        double t2 = now();
        if (pitched()) return 1;
        double t3 = now();
        CK(cudaHostUnregister(host.data()));
        double t4 = now();
        std::printf("pitched %.2f ms | register %.2f + copy %.2f + unregister %.2f ms\n", 1e3 * (t1 - t0),
                    1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3));
    }
    // staged: chunks of C planes, packed, double-buffered pinned staging, T host threads scatter
    const int C = 16;
    float* stg[2];
    CK(cudaHostAlloc(&stg[0], size_t(C) * n * n * 4, cudaHostAllocDefault));
    CK(cudaHostAlloc(&stg[1], size_t(C) * n * n * 4, cudaHostAllocDefault));
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    for (int T : {1, 2, 4, 8}) {
        double best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            double t0 = now();
            const int nch = n / C;
            CK(cudaMemcpyAsync(stg[0], d, size_t(C) * n * n * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaEventRecord(ev[0], s));
            for (int c = 0; c < nch; ++c) {
                const int b = c & 1;
                if (c + 1 < nch) {
                    CK(cudaMemcpyAsync(stg[b ^ 1], d + size_t(c + 1) * C * n * n, size_t(C) * n * n * 4,
                                       cudaMemcpyDeviceToHost, s));
                    CK(cudaEventRecord(ev[b ^ 1], s));
                }
                CK(cudaEventSynchronize(ev[b]));
                std::vector<std::thread> th;
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&, t] {
                        for (int r = t; r < C * n; r += T) {  // row r of the chunk: plane r / n, row r % n
                            const int x = c * C + r / n, y = r % n;
                            std::memcpy(&host[(size_t(x + halo) * np + y + halo) * np + halo],
                                        stg[b] + size_t(r) * n, 4 * n);
                        }
                    });
                for (auto& x : th) x.join();
            }
            best = std::min(best, now() - t0);
        }
        std::printf("staged C=%d T=%d %.2f ms\n", C, T, 1e3 * best);
    }
    return 0;
}
