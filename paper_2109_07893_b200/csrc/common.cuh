// Shared helpers for the sm_100a kernels of libdgnn_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dgnn_b200.h"

namespace dgnn {

void set_error(const char* fmt, ...);
// Counts every kernel launch made through the C ABI (dgnn_launch_count).
void note_launch();
// Checks cudaGetLastError after a launch sequence.
int launch_status(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int kMaxSMs = 192;  // static bound for device-side arrays; launches use num_sms()
// multiprocessors of the current device (queried once per device; 148 on B200)
int num_sms();
// CTAs of the persistent (one CTA per SM) kernels: num_sms() minus the SMs kept
// free for concurrent communication kernels (dgnn_set_sm_reserve)
int persistent_ctas();

// ---- frames -------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T* frame_row(const dgnn_frame& f, int64_t i) {
    if (f.rows_per_slab <= 0) return reinterpret_cast<T*>(f.ptr) + i * f.ld;
    // row indices are vertex ids (< 2^31): a 32-bit division, several times
    // cheaper than the 64-bit one on the gather path of the owner layout
    const uint32_t rps = (uint32_t)f.rows_per_slab;
    const int64_t s = (uint32_t)i / rps;
    const int64_t r = (uint32_t)i - (uint32_t)s * rps;
    return reinterpret_cast<T*>(f.ptr) + s * f.slab_stride + r * f.ld;
}

// ---- hub rows of the aggregation ----------------------------------------
// Rows with more than kHubRow stored entries (heavy-tailed graphs: hub
// accounts) are skipped by the per-row gather loops of the SpMM / K3
// kernels (one lane group would walk them serially while the whole tile
// waits) and computed afterwards by hub_rows_kernel (spmm.cu): a CTA per hub
// row, edges split over lane groups, partials reduced in a fixed tree --
// deterministic, and the same for the tcgen05 and SIMT instances.
constexpr int kHubRow = 16;   // c3 (heavy-tailed): 64 left most 128-row tiles holding a 17..64-entry row as a serial tail (median tile max degree 21)

// ---- tile-blocked layout of the LSTM step caches -----------------------
// The per-step cell state c, the gate cache (overwritten in place by dz) and
// the cell-state gradient dc are stored "tile-blocked": rows in tiles of 128,
// columns in groups of 4, and each (tile, group) block -- 4 floats of the
// tile's rows -- contiguous.  Every producer and consumer of these caches
// holds one row per lane, so a warp's float4 access covers 512 contiguous
// bytes instead of 32 rows x 16 B.  Compact: the last tile of a step only
// holds its own rows, so a step of n rows x W floats occupies n W floats.
// (h stays row-major: the next layer gathers it by vertex.)
__host__ __device__ __forceinline__ int64_t tb_off(int64_t row, int col, int w, int64_t n) {
    const int64_t t0 = row & ~(int64_t)127;
    const int64_t tr = n - t0 < 128 ? n - t0 : 128;
    return t0 * w + (int64_t)(col >> 2) * 4 * tr + (row - t0) * 4 + (col & 3);
}

// ---- warp helpers -------------------------------------------------------
__device__ __forceinline__ int warp_inclusive_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// LSTM gate activations, shared by every LSTM kernel (SIMT, tensor-core,
// warp-specialised) so their results stay bitwise equal.  sigmoid: MUFU
// ex2/rcp, a few ulp relative.  tanh: for |x| < 0.6 an odd minimax
// polynomial x + x^3 Q(x^2) (<= 0.6 ulp relative in fp32, fitted on
// [0, 0.6]) -- the 2 sigmoid(2x) - 1 form loses all relative accuracy near
// 0 (~2.4e-7 absolute), which after a few dozen recurrent steps showed up as
// ~1.6e-6 absolute error in near-zero embeddings at configs[1]; for
// |x| >= 0.6, 1 - 2 / (1 + e^{2|x|}) with the sign restored (MUFU, ~3e-7
// relative).
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float act_sigmoid(float x) { return rcp_approx(1.0f + ex2_approx(-1.4426950408889634f * x)); }
__device__ __forceinline__ float act_tanh(float x) {
    const float ax = fabsf(x);
    const float u = x * x;
    float q = fmaf(-0.005984960589557886f, u, 0.020868148654699326f);
    q = fmaf(q, u, -0.053803566843271255f);
    q = fmaf(q, u, 0.13332132995128632f);
    q = fmaf(q, u, -0.3333330452442169f);
    const float small = fmaf(x * u, q, x);
    const float big = fmaf(-2.0f, rcp_approx(1.0f + ex2_approx(2.885390081777927f * ax)), 1.0f);
    return ax < 0.6f ? small : copysignf(big, x);
}

// device-wide exclusive scan (in place), implemented in graph.cu
size_t scan_workspace_bytes(int64_t n);
int exclusive_scan_i32(int32_t* data, int64_t n, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace dgnn

#define DGNN_CHECK_ARG(cond, msg)                 \
    do {                                          \
        if (!(cond)) {                            \
            ::dgnn::set_error("%s", msg);         \
            return DGNN_EINPUT;                   \
        }                                         \
    } while (0)
