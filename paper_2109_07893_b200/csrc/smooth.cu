// M-smoothing of the snapshot sequence on the device (TM-GCN preprocessing,
// SURVEY §8f.1): smoothed A~_t = sum_k M[t,k] A_k over the window, i.e.
// `m_transform_graph` -> `sparse_weighted_sum` (dtdg.py:239-252,
// core.py:173-192) for window 2: a weighted union of two canonical CSRs.
//
// The reference concatenates the terms in ascending k and canonicalises with
// np.add.at from zeros, so an entry present in both gets
// fl(fl(wa a) + fl(wb b)) and an entry present in one gets fl(w v) (0 + x is
// exact); computed here with __dmul_rn / __dadd_rn (no FMA contraction), the
// values are bit-identical.  Entries whose sum is exactly 0 would be dropped
// by the reference; with non-negative weights and positive raw values (the
// only case the engine smooths on the device) none can occur.
//
// Every entry is handled by its own thread (no per-row loops, so hub rows
// of heavy-tailed graphs cost nothing extra):
//   1. flag B entries absent from A's row (binary search; an entry's row is
//      found by galloping from an interpolation guess);
//   2. exclusive scan of the flags (S);
//   3. row counts |A_r| + |B_r \ A_r| -> exclusive scan -> out rowptr;
//   4. A entries: position = out_rowptr[r] + rank in A_r + #(B_r \ A_r < e),
//      the last term S[lower_bound_B(e)] - S[rowstart_B];
//   5. B \ A entries: position = out_rowptr[r] + #(A_r < e) + S[j] - S[rowstart_B].

#include "common.cuh"

namespace dgnn {
namespace {

// same row, found from an interpolation guess e * n / nnz by galloping
// (a few dependent loads instead of log2 n for every entry)
__device__ __forceinline__ int32_t row_of_guess(const int32_t* __restrict__ rp, int32_t n, int64_t nnz, int64_t e) {
    int32_t r = (int32_t)min((int64_t)n - 1, e * (int64_t)n / nnz);
    int32_t lo, hi;                       // rp[lo] <= e < rp[hi]
    if (rp[r] > e) {
        hi = r;
        int32_t step = 1;
        lo = r - 1;
        while (lo > 0 && rp[lo] > e) {
            hi = lo;
            step <<= 1;
            lo = r - step > 0 ? r - step : 0;
        }
    } else {
        lo = r;
        int32_t step = 1;
        hi = r + 1;
        while (hi < n && rp[hi] <= e) {
            lo = hi;
            step <<= 1;
            hi = r + step < n ? r + step : n;
        }
    }
    while (lo + 1 < hi) {
        const int32_t mid = (int32_t)(((int64_t)lo + hi) >> 1);
        if (rp[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t lower_bound(const int32_t* __restrict__ a, int64_t lo, int64_t hi, int32_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void flag_b_not_in_a(int32_t n, int64_t nnz_b, const int32_t* __restrict__ rp_a,
                                const int32_t* __restrict__ col_a, const int32_t* __restrict__ rp_b,
                                const int32_t* __restrict__ col_b, int32_t* __restrict__ flag) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz_b; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = row_of_guess(rp_b, n, nnz_b, j);
        const int32_t e = col_b[j];
        const int64_t a1 = rp_a[r + 1];
        const int64_t p = lower_bound(col_a, rp_a[r], a1, e);
        flag[j] = (p < a1 && col_a[p] == e) ? 0 : 1;
    }
}

__global__ void merged_counts(int32_t n, const int32_t* __restrict__ rp_a, const int32_t* __restrict__ rp_b,
                              const int32_t* __restrict__ scan_b, int32_t* __restrict__ out_rowptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n; r += (int64_t)gridDim.x * blockDim.x) {
        out_rowptr[r] = r < n ? (rp_a[r + 1] - rp_a[r]) + (scan_b[rp_b[r + 1]] - scan_b[rp_b[r]]) : 0;
    }
}

__global__ void write_a(int32_t n, int64_t nnz_a, const int32_t* __restrict__ rp_a, const int32_t* __restrict__ col_a,
                        const double* __restrict__ val_a, double wa, const int32_t* __restrict__ rp_b,
                        const int32_t* __restrict__ col_b, const double* __restrict__ val_b, double wb,
                        const int32_t* __restrict__ scan_b, const int32_t* __restrict__ out_rowptr,
                        int32_t* __restrict__ out_col, double* __restrict__ out_val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz_a; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = row_of_guess(rp_a, n, nnz_a, i);
        const int32_t e = col_a[i];
        const int64_t b0 = rp_b[r], b1 = rp_b[r + 1];
        const int64_t lb = lower_bound(col_b, b0, b1, e);
        const bool match = lb < b1 && col_b[lb] == e;
        const int64_t pos = out_rowptr[r] + (i - rp_a[r]) + (scan_b[lb] - scan_b[b0]);
        double v = __dmul_rn(wa, val_a ? val_a[i] : 1.0);
        if (match) v = __dadd_rn(v, __dmul_rn(wb, val_b ? val_b[lb] : 1.0));
        out_col[pos] = e;
        out_val[pos] = v;
    }
}

__global__ void write_b_only(int32_t n, int64_t nnz_b, const int32_t* __restrict__ rp_a,
                             const int32_t* __restrict__ col_a, const int32_t* __restrict__ rp_b,
                             const int32_t* __restrict__ col_b, const double* __restrict__ val_b, double wb,
                             const int32_t* __restrict__ flag, const int32_t* __restrict__ scan_b,
                             const int32_t* __restrict__ out_rowptr, int32_t* __restrict__ out_col,
                             double* __restrict__ out_val) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nnz_b; j += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[j]) continue;
        const int32_t r = row_of_guess(rp_b, n, nnz_b, j);
        const int32_t e = col_b[j];
        const int64_t a0 = rp_a[r];
        const int64_t la = lower_bound(col_a, a0, rp_a[r + 1], e) - a0;
        const int64_t pos = out_rowptr[r] + la + (scan_b[j] - scan_b[rp_b[r]]);
        out_col[pos] = e;
        out_val[pos] = __dmul_rn(wb, val_b ? val_b[j] : 1.0);
    }
}

int grid_for(int64_t items) {
    int64_t g = cdiv(items, 256);
    const int64_t cap = 8LL * num_sms();
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace
}  // namespace dgnn

extern "C" {

size_t dgnn_csr_weighted_merge_workspace(int32_t n, int64_t nnz_b) {
    const int64_t flags = (nnz_b + 1 + 63) / 64 * 64;
    const int64_t big = nnz_b + 1 > (int64_t)n + 1 ? nnz_b + 1 : (int64_t)n + 1;
    return (size_t)flags * 2 * sizeof(int32_t) + dgnn::scan_workspace_bytes(big) + 256;
}

int dgnn_csr_weighted_merge(int32_t n, const int32_t* rp_a, const int32_t* col_a, const double* val_a, int64_t nnz_a,
                            double wa, const int32_t* rp_b, const int32_t* col_b, const double* val_b, int64_t nnz_b,
                            double wb, int32_t* out_rowptr, int32_t* out_col, double* out_val, int64_t out_cap,
                            void* ws, size_t ws_bytes, void* stream) {
    using namespace dgnn;
    DGNN_CHECK_ARG(n >= 0 && nnz_a >= 0 && nnz_b >= 0, "negative size");
    DGNN_CHECK_ARG(out_cap >= nnz_a + nnz_b, "merged capacity below nnz_a + nnz_b");
    DGNN_CHECK_ARG(ws_bytes >= dgnn_csr_weighted_merge_workspace(n, nnz_b), "merge workspace too small");
    cudaStream_t st = as_stream(stream);
    const int64_t flags_len = (nnz_b + 1 + 63) / 64 * 64;
    int32_t* flag = reinterpret_cast<int32_t*>(ws);
    int32_t* scan_b = flag + flags_len;
    void* sws = scan_b + flags_len;
    const size_t sws_bytes = ws_bytes - (size_t)flags_len * 2 * sizeof(int32_t);
    if (nnz_b) {
        note_launch();
        flag_b_not_in_a<<<grid_for(nnz_b), 256, 0, st>>>(n, nnz_b, rp_a, col_a, rp_b, col_b, flag);
        cudaMemcpyAsync(scan_b, flag, nnz_b * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
    }
    cudaMemsetAsync(scan_b + nnz_b, 0, sizeof(int32_t), st);
    int rc = exclusive_scan_i32(scan_b, nnz_b + 1, sws, sws_bytes, st);
    if (rc) return rc;
    note_launch();
    merged_counts<<<grid_for((int64_t)n + 1), 256, 0, st>>>(n, rp_a, rp_b, scan_b, out_rowptr);
    rc = exclusive_scan_i32(out_rowptr, (int64_t)n + 1, sws, sws_bytes, st);
    if (rc) return rc;
    if (nnz_a) {
        note_launch();
        write_a<<<grid_for(nnz_a), 256, 0, st>>>(n, nnz_a, rp_a, col_a, val_a, wa, rp_b, col_b, val_b, wb, scan_b,
                                                 out_rowptr, out_col, out_val);
    }
    if (nnz_b) {
        note_launch();
        write_b_only<<<grid_for(nnz_b), 256, 0, st>>>(n, nnz_b, rp_a, col_a, rp_b, col_b, val_b, wb, flag, scan_b,
                                                      out_rowptr, out_col, out_val);
    }
    return launch_status("dgnn_csr_weighted_merge");
}

}  // extern "C"
