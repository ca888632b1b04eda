// head_scatter (dz seeds of the head) at the configs[1] shape: N = 750k
// vertices, E = 64, 2 classes, ~190k labelled pairs per step (uniform
// endpoints); lanes per vertex / grid size from the build.
// Build/run: scripts/head_probe.sh
#include "../paper_2109_07893_b200/csrc/head.cu"
#ifndef HP_C3
#define HP_C3 0
#endif
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cmath>

int main() {
    // HP_C3: the configs[2] shape (1M vertices, E = 32, 400k pairs per step,
    // heavy-tailed endpoints: x = n u^2.2, ~1.5k slots on the top vertex as
    // in the configs[2] label sets)
    const int n = HP_C3 ? 1000000 : 750000, C = 2;
    constexpr int ep = HP_C3 ? 32 : 64;
    const int64_t npairs = HP_C3 ? 400000 : 190000;
    std::mt19937 g(1);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<std::pair<int, int>> inc;
    for (int64_t p = 0; p < npairs; ++p)
        for (int side = 0; side < 2; ++side) {
            const double u = U(g);
            const int x = HP_C3 ? std::min(n - 1, (int)(n * std::pow(u, 2.2))) : (int)(g() % n);
            inc.push_back({x, (int)(2 * p + side)});
        }
    std::sort(inc.begin(), inc.end());
    std::vector<int> ptr(n + 1, 0), slot(inc.size());
    for (size_t i = 0; i < inc.size(); ++i) { ptr[inc[i].first + 1]++; slot[i] = inc[i].second; }
    for (int i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
    int *dptr, *dslot; double* dl; float *hw, *dz;
    cudaMalloc(&dptr, (n + 1) * 4); cudaMalloc(&dslot, inc.size() * 4); cudaMalloc(&dl, npairs * C * 8);
    cudaMalloc(&hw, 2 * ep * C * 4); cudaMalloc(&dz, (size_t)n * ep * 4);
    cudaMemcpy(dptr, ptr.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dslot, slot.data(), inc.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dl, 0, npairs * C * 8); cudaMemset(hw, 0, 2 * ep * C * 4);
    dgnn_frame f{dz, ep, 0, 0};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) dgnn::head_scatter_t<ep>(n, dptr, dslot, dl, hw, C, f, 0);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int it = 0; it < reps; ++it) dgnn::head_scatter_t<ep>(n, dptr, dslot, dl, hw, C, f, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaEventRecord(e0);
    for (int it = 0; it < reps; ++it) cudaMemsetAsync(dz, 0, (size_t)n * ep * 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    std::vector<int> act;
    for (int x = 0; x < n; ++x) if (ptr[x + 1] > ptr[x]) act.push_back(x);
#ifdef HP_SORT
    // active vertices by decreasing incidence count (ties by index)
    std::stable_sort(act.begin(), act.end(), [&](int a, int b) { return ptr[a + 1] - ptr[a] > ptr[b + 1] - ptr[b]; });
#endif
    int* dact; cudaMalloc(&dact, act.size() * 4);
    cudaMemcpy(dact, act.data(), act.size() * 4, cudaMemcpyHostToDevice);
    for (int it = 0; it < 3; ++it) dgnn::head_scatter_t<ep>(n, dptr, dslot, dl, hw, C, f, 0, (int)act.size(), dact);
    cudaEventRecord(e0);
    for (int it = 0; it < reps; ++it) dgnn::head_scatter_t<ep>(n, dptr, dslot, dl, hw, C, f, 0, (int)act.size(), dact);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms3; cudaEventElapsedTime(&ms3, e0, e1);
    printf("head_scatter GL=%d GLA=%d BLK=%d  all %.1f us  active (%zu of %d) %.1f us  (memset of dz %.1f us)  err=%s\n",
           DGNN_HS_GL, DGNN_HS_GLA, DGNN_HS_BLK, 1e3 * ms / reps, act.size(), n, 1e3 * ms3 / reps, 1e3 * ms2 / reps,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
