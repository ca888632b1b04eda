// exclusive_scan_i32 against a host scan for several sizes (incl. partial tiles).
// Build/run: nvcc ... scripts/scan_test.cu -Lpaper_2109_07893_b200 -ldgnn_b200 (scripts/scan_test.sh)
#include "../paper_2109_07893_b200/csrc/common.cuh"
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

int main() {
    const long sizes[] = {1, 5, 4096, 4097, 100000, 1000001, 10000001};
    int bad = 0;
    for (long n : sizes) {
        std::vector<int> h(n), r(n);
        for (long i = 0; i < n; ++i) h[i] = (int)((i * 2654435761u) % 7);
        int* d; cudaMalloc(&d, n * 4); cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
        size_t wb = dgnn::scan_workspace_bytes(n);
        void* ws; cudaMalloc(&ws, wb);
        int rc = dgnn::exclusive_scan_i32(d, n, ws, wb, 0);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(r.data(), d, n * 4, cudaMemcpyDeviceToHost);
        long run = 0, wrong = 0;
        for (long i = 0; i < n; ++i) { if (r[i] != (int)run) ++wrong; run += h[i]; }
        printf("n=%ld rc=%d err=%s wrong=%ld\n", n, rc, cudaGetErrorString(e), wrong);
        bad += wrong != 0 || e != cudaSuccess;
        cudaFree(d); cudaFree(ws);
    }
    return bad;
}
