// Backward LSTM step kernel (K6) at configs[1] shapes (rows 750k, hp 64, kx
// from argv), producer warp count from the build (-DDGNN_BWD_NPROD).
// Build/run: scripts/bwd_roles.sh
#include "../paper_2109_07893_b200/csrc/lstm_ws.cu"
#include <cstdio>

int main(int argc, char** argv) {
    const int64_t rows = 750000;
    const int kx = argc > 1 ? atoi(argv[1]) : 128, hp = 64, N = 4 * hp;
    float *dy, *dhi, *dci, *gates, *cp, *cn, *img, *dx, *dho, *dco;
    cudaMalloc(&dy, rows * hp * 4); cudaMalloc(&dhi, rows * hp * 4); cudaMalloc(&dci, rows * hp * 4);
    cudaMalloc(&gates, rows * N * 4); cudaMalloc(&cp, rows * hp * 4); cudaMalloc(&cn, rows * hp * 4);
    cudaMalloc(&img, 64 << 20); cudaMalloc(&dx, rows * kx * 4); cudaMalloc(&dho, rows * hp * 4);
    cudaMalloc(&dco, rows * hp * 4);
    for (float* p : {dy, dhi, dci, cp, cn, dho, dco}) cudaMemset(p, 0, rows * hp * 4);
    cudaMemset(gates, 0, rows * N * 4); cudaMemset(img, 0, 64 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) dgnn::lstm_bwd_ws_t<64>(rows, kx, dy, dhi, dci, gates, cp, cn, img, dx, kx, dho, dco, 0);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int it = 0; it < reps; ++it) dgnn::lstm_bwd_ws_t<64>(rows, kx, dy, dhi, dci, gates, cp, cn, img, dx, kx, dho, dco, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 4.0 * rows * (4 * hp + 4 * hp + 4 * hp + kx + 2 * hp);
    printf("bwd nprod=%d kx=%d  %.1f us/launch  %.0f GB/s algorithmic  err=%s\n", DGNN_BWD_NPROD, kx, 1e3 * ms / reps,
           bytes / (ms / reps * 1e6), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
