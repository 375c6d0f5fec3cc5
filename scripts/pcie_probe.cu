// PCIe probe: H2D / D2H alone and concurrent, 1D vs 2D copies, cudaHostAlloc
// vs cudaHostRegister, whole buffer vs 5 MB chunks.
// nvcc -O2 -o build/pcie_probe scripts/pcie_probe.cu && build/pcie_probe
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    const size_t n = size_t(256) << 20;
    char *ha, *hb, *da, *db;
    cudaHostAlloc(&ha, n, 0); cudaHostAlloc(&hb, n, 0);
    char* hr = (char*)aligned_alloc(4096, n); char* hr2 = (char*)aligned_alloc(4096, n);
    for (size_t i = 0; i < n; i += 4096) { hr[i] = 1; hr2[i] = 1; ha[i] = 1; hb[i] = 1; }
    cudaHostRegister(hr, n, cudaHostRegisterPortable); cudaHostRegister(hr2, n, cudaHostRegisterPortable);
    cudaMalloc(&da, n); cudaMalloc(&db, n);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    auto run = [&](const char* name, auto f) {
        double best = 1e9;
        for (int r = 0; r < 3; ++r) { cudaDeviceSynchronize(); double t0 = now(); f(); cudaDeviceSynchronize(); best = std::min(best, now() - t0); }
        return best;
    };
    for (int reg = 0; reg < 2; ++reg) {
        char* h1 = reg ? hr : ha; char* h2 = reg ? hr2 : hb;
        for (size_t chunk : {n, size_t(5) << 20, size_t(1) << 20}) {
            auto h2d = [&] { for (size_t o = 0; o < n; o += chunk) cudaMemcpyAsync(da + o, h1 + o, chunk, cudaMemcpyHostToDevice, s1); };
            auto d2h = [&] { for (size_t o = 0; o < n; o += chunk) cudaMemcpyAsync(h2 + o, db + o, chunk, cudaMemcpyDeviceToHost, s2); };
            double a = run("h2d", h2d), b = run("d2h", d2h), c = run("both", [&] { h2d(); d2h(); });
            // 2D: 4 rows of chunk/4 with pitch n/4 (an SoA chunk of 4 components)
            auto h2d2 = [&] { size_t w = chunk / 4, p = n / 4; for (size_t o = 0; o < p; o += w) cudaMemcpy2DAsync(da + o, p, h1 + o, p, w, 4, cudaMemcpyHostToDevice, s1); };
            auto d2h2 = [&] { size_t w = chunk / 4, p = n / 4; for (size_t o = 0; o < p; o += w) cudaMemcpy2DAsync(h2 + o, p, db + o, p, w, 4, cudaMemcpyDeviceToHost, s2); };
            double a2 = run("h2d2", h2d2), b2 = run("d2h2", d2h2), c2 = run("both2", [&] { h2d2(); d2h2(); });
            printf("%s chunk %6zu KB: 1D H2D %5.1f D2H %5.1f both %5.1f GB/s | 2D H2D %5.1f D2H %5.1f both %5.1f GB/s\n",
                   reg ? "registered" : "hostalloc ", chunk >> 10, n / a / 1e9, n / b / 1e9, 2 * n / c / 1e9,
                   n / a2 / 1e9, n / b2 / 1e9, 2 * n / c2 / 1e9);
        }
    }
    return 0;
}
