// Bottleneck probe for the TMEM-operand weight-gradient kernel (dw_ts.cu):
// bench-shaped launch (rows 8 x 750k, hp 64, kx from argv) with parts
// disabled (DGNN_DTS_PROBE).  Build/run: scripts/dts_probe.sh
#include "../paper_2109_07893_b200/csrc/dw_ts.cu"
#include <cstdio>

int main(int argc, char** argv) {
    const int64_t np = 750000, rows = 8 * np;
    const int kx = argc > 1 ? atoi(argv[1]) : 128, hp = 64, M = 4 * hp;
    float *x, *y, *h0, *dz;
    double *gw, *gb;
    cudaMalloc(&x, rows * kx * 4); cudaMalloc(&y, rows * hp * 4); cudaMalloc(&h0, np * hp * 4);
    cudaMalloc(&dz, rows * M * 4); cudaMalloc(&gw, (kx + hp) * M * 8); cudaMalloc(&gb, M * 8);
    cudaMemset(x, 0, rows * kx * 4); cudaMemset(y, 0, rows * hp * 4); cudaMemset(h0, 0, np * hp * 4);
    cudaMemset(dz, 0, rows * M * 4);
    const size_t wsb = dgnn_lstm_weight_grad_tc_workspace(kx, hp);
    void* ws; cudaMalloc(&ws, wsb);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    dgnn::lstm_dw_ts_t<64>(rows, np, kx, x, kx, y, h0, dz, gw, gb, ws, wsb, 0);
    cudaEventRecord(e0);
    const int reps = 3;
    for (int it = 0; it < reps; ++it) dgnn::lstm_dw_ts_t<64>(rows, np, kx, x, kx, y, h0, dz, gw, gb, ws, wsb, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)rows * (M + kx + hp) * 4;
    printf("dts probe=%d kx=%d  %.1f us/launch  %.0f GB/s algorithmic  err=%s\n", DGNN_DTS_PROBE, kx,
           1e3 * ms / reps, bytes / (ms / reps * 1e6), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
