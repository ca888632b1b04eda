// Bottleneck probe for the warp-specialised forward LSTM kernel: times the
// bench-shaped launch (rows 750k, kx 64, hp 64) with parts of the pipeline
// disabled (see DGNN_WS_PROBE in lstm_ws.cu).  Build: scripts/ws_probe.sh
#include "../paper_2109_07893_b200/csrc/lstm_ws.cu"
#include <cstdio>
#include <vector>
#ifndef HPP
#define HPP 64
#endif

int main(int argc, char** argv) {
    const int64_t rows = 750000;
    const int kx = argc > 1 ? atoi(argv[1]) : 64, N = 4 * HPP;
    const int hp = HPP;
    float *x, *h, *c, *img, *b, *ho, *co, *gates;
    cudaMalloc(&x, rows * kx * 4); cudaMalloc(&h, rows * hp * 4); cudaMalloc(&c, rows * hp * 4);
    cudaMalloc(&ho, rows * hp * 4); cudaMalloc(&co, rows * hp * 4); cudaMalloc(&gates, rows * N * 4);
    cudaMalloc(&img, 64 << 20); cudaMalloc(&b, N * 4);
    cudaMemset(x, 0, rows * kx * 4); cudaMemset(h, 0, rows * hp * 4); cudaMemset(c, 0, rows * hp * 4);
    cudaMemset(img, 0, 64 << 20); cudaMemset(b, 0, N * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) dgnn::lstm_fwd_ws_t<HPP>(rows, kx, x, kx, h, c, img, b, ho, co, gates, 0);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int it = 0; it < reps; ++it) dgnn::lstm_fwd_ws_t<HPP>(rows, kx, x, kx, h, c, img, b, ho, co, gates, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)rows * (kx + hp + hp + hp + hp + N) * 4;
    printf("probe=%d kx=%d  %.1f us/launch  %.0f GB/s algorithmic  err=%s\n", DGNN_WS_PROBE, kx, 1e3 * ms / reps,
           bytes / (ms / reps * 1e6), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
