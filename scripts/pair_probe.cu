// Bottleneck probe for the CTA-pair forward LSTM kernel (lstm_pair.cu): times
// the configs[1] layer-1 launch (rows 750k, kx, hp 64, no gate cache) with
// parts of the pipeline disabled (DGNN_PAIR_PROBE).  Build: scripts/pair_probe.sh
#include "../paper_2109_07893_b200/csrc/lstm_pair.cu"
#include <cstdio>

int main(int argc, char** argv) {
    const int64_t rows = 750000;
    const int kx = argc > 1 ? atoi(argv[1]) : 128, hp = 64, N = 4 * hp;
    const int keep = argc > 2 ? atoi(argv[2]) : 0;
    float *x, *h, *c, *img, *b, *ho, *co, *gates;
    cudaMalloc(&x, rows * kx * 4); cudaMalloc(&h, rows * hp * 4); cudaMalloc(&c, rows * hp * 4);
    cudaMalloc(&ho, rows * hp * 4); cudaMalloc(&co, rows * hp * 4); cudaMalloc(&gates, rows * N * 4);
    cudaMalloc(&img, 64 << 20); cudaMalloc(&b, N * 4);
    cudaMemset(x, 0, rows * kx * 4); cudaMemset(h, 0, rows * hp * 4); cudaMemset(c, 0, rows * hp * 4);
    cudaMemset(img, 0, 64 << 20); cudaMemset(b, 0, N * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float* g = keep ? gates : nullptr;
    for (int it = 0; it < 3; ++it) dgnn::lstm_fwd_pair_t<64>(rows, kx, x, kx, h, c, img, b, ho, co, g, 0);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int it = 0; it < reps; ++it) dgnn::lstm_fwd_pair_t<64>(rows, kx, x, kx, h, c, img, b, ho, co, g, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("pair probe=%2d kx=%d keep=%d  %.1f us/launch  err=%s\n", DGNN_PAIR_PROBE, kx, keep, 1e3 * ms / reps,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
