// GCN weight-gradient kernel at the configs[1] shape (N = 750k, F = H = 64,
// skip cell) with the loader / converter warp counts from the command line
// build (-DDGNN_GDW_NLOAD / -DDGNN_GDW_NCONV).  Build/run: scripts/gdw_probe.sh
#include "../paper_2109_07893_b200/csrc/gcn_dw_tc.cu"
#include <cstdio>

int main() {
    const int n = 750000, fp = 64, hp = 64, rw = fp + hp;
    float *s, *dr, *r;
    double* gw;
    cudaMalloc(&s, (size_t)n * fp * 4); cudaMalloc(&dr, (size_t)n * rw * 4); cudaMalloc(&r, (size_t)n * rw * 4);
    cudaMalloc(&gw, fp * hp * 8);
    cudaMemset(s, 0, (size_t)n * fp * 4); cudaMemset(dr, 0, (size_t)n * rw * 4); cudaMemset(r, 0, (size_t)n * rw * 4);
    const size_t wsb = dgnn::gcn_dw_tc_workspace(fp, hp);
    void* ws; cudaMalloc(&ws, wsb);
    dgnn_frame fs{s, fp, 0, 0}, fdr{dr, rw, 0, 0}, fr{r, rw, 0, 0};
    // a 1 GB buffer written between launches keeps the operands out of L2
    char* flush; cudaMalloc(&flush, 1 << 30);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0.f;
    const int reps = 10;
    for (int it = 0; it <= reps; ++it) {
        cudaMemsetAsync(flush, it, 1 << 30);
        cudaEventRecord(e0);
        dgnn::gcn_dw_tc(n, fs, fdr, fr, fp, hp, 1, gw, ws, wsb, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (it) tot += ms;
    }
    const double bytes = 4.0 * n * (fp + 2 * hp);
    printf("gdw nload=%d nconv=%d  %.1f us  %.0f GB/s  err=%s\n", DGNN_GDW_NLOAD, DGNN_GDW_NCONV, 1e3 * tot / reps,
           bytes / (tot / reps * 1e6), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
