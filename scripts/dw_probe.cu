// Bottleneck probe for the weight-gradient kernel: bench-shaped launch
// (rows 8 x 750k, np 750k, hp 64, kx from argv) with parts disabled (see
// DGNN_DW_PROBE in dw_tc.cu).  Build/run: scripts/dw_probe.sh
#include "../paper_2109_07893_b200/csrc/dw_tc.cu"
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
    dgnn::lstm_dw_tc_t<64>(rows, np, kx, x, kx, y, h0, dz, gw, gb, ws, wsb, 0);
    cudaEventRecord(e0);
    const int reps = 3;
    for (int it = 0; it < reps; ++it) dgnn::lstm_dw_tc_t<64>(rows, np, kx, x, kx, y, h0, dz, gw, gb, ws, wsb, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)rows * (M + kx + hp) * 4;
#if DGNN_DW_PROBE & 16
    {
        unsigned long long prof[dgnn::kMaxSMs * 8];
        const int nsm = dgnn::num_sms();
        cudaMemcpyFromSymbol(prof, dgnn::dw_prof, sizeof(prof));
        double f[6] = {0, 0, 0, 0, 0, 0};
        for (int c = 0; c < nsm; ++c)
            for (int k = 0; k < 6; ++k) f[k] += (double)prof[c * 8 + k] / nsm;
        printf("cycles/CTA %.0f: loader wait-empty %.1f%%  converter wait-landed %.1f%%  mma wait-full %.1f%%  "
               "mma wait-accempty %.1f%%  epilogue wait-accfull %.1f%%\n", f[5], 100 * f[0] / f[5], 100 * f[1] / f[5],
               100 * f[2] / f[5], 100 * f[3] / f[5], 100 * f[4] / f[5]);
    }
#endif
    printf("dw probe=%d kx=%d  %.1f us/launch  %.0f GB/s algorithmic  err=%s\n", DGNN_DW_PROBE, kx, 1e3 * ms / reps,
           bytes / (ms / reps * 1e6), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
