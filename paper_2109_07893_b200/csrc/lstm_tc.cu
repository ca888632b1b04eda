// Temporal stage on the 5th-generation tensor cores (K5): the LSTM gate GEMM
// z = [x | h_prev] W + b runs as tcgen05.mma kind::tf32 with the 3xTF32
// split (fp32-accurate), accumulator in TMEM; the cell update (sigmoid/tanh,
// c = f c_prev + i g, h = o tanh c) is the epilogue, fed by tcgen05.ld, so z
// never touches HBM.  Reference: training.py:370-391.
//
// CTA = 128 vertex rows x all 4*HP gate columns (one M=128, N=4*HP MMA
// shape; HP=128 issues two N=256 halves).  K is streamed in chunks of 16
// fp32 through a 2-stage shared-memory ring: every thread stages the
// activation chunk (global fp32 -> hi/lo tf32 split -> SW64 tile) and copies
// the pre-split, pre-swizzled weight chunk; one thread issues the MMAs and
// commits them to the stage's mbarrier, so staging of chunk c+1 overlaps the
// MMAs of chunk c.  Two CTAs fit per SM (96 KB smem, <= 256 TMEM columns
// each for HP <= 64), overlapping one CTA's epilogue with the other's MMAs.
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

constexpr int TC_BM = 128;
constexpr int TC_KC = 16;  // fp32 K-elements per staged chunk (one SW64 row)

// Weight image for the B operand: [chunk][hi|lo][N rows][16 fp32], each
// [N][16] block an SW64 tile (byte-identical to its shared-memory copy).
// Source w is N x K row-major (K-major), leading dimension ldw.
__global__ void wimg_kernel(int N, int K, const float* __restrict__ w, int64_t ldw, float* __restrict__ img) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int nch = (K + TC_KC - 1) / TC_KC;
    if (i >= (int64_t)nch * N * 4) return;
    const int q = (int)(i & 3);
    const int n = (int)((i >> 2) % N);
    const int ch = (int)(i / (4 * (int64_t)N));
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int k = ch * TC_KC + 4 * q + j;
        v[j] = k < K ? w[(int64_t)n * ldw + k] : 0.f;
    }
    float4 hi, lo;
    split4(make_float4(v[0], v[1], v[2], v[3]), hi, lo);
    char* base = reinterpret_cast<char*>(img) + (size_t)ch * 2 * N * 64;
    *reinterpret_cast<float4*>(base + sw64(n, q)) = hi;
    *reinterpret_cast<float4*>(base + (size_t)N * 64 + sw64(n, q)) = lo;
}

// ---------------------------------------------------------------------------
// shared mainloop: D[128 x N] (TMEM) = A[128 x K] * B[N x K]^T, 3xTF32

struct StageLayout {
    uint32_t a_hi, a_lo, b;   // smem addresses (b: [hi | lo] copy of the image chunk)
};

template <int N>
struct TcCfg {
    static constexpr int A_BYTES = TC_BM * 64;      // one SW64 tile of 128 rows
    static constexpr int B_BYTES = 2 * N * 64;      // hi + lo tiles of N rows
    static constexpr int STAGE = 2 * A_BYTES + B_BYTES;
    static constexpr int SMEM = 2 * STAGE + 1024 + 64;
    static constexpr int TMEM_COLS = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : (N <= 256 ? 256 : 512)));
    static constexpr int MMA_N = N > 256 ? 256 : N;
};

// Stage one K chunk: A via `load4(r, k)` (returns the 4 fp32 at row r, k..k+3),
// B by copying the image chunk.
template <int N, class LoadA>
__device__ __forceinline__ void stage_chunk(const StageLayout& s, int ch, const float* __restrict__ img,
                                            LoadA load4) {
    const int tid = threadIdx.x;
    for (int idx = tid; idx < TC_BM * 4; idx += blockDim.x) {
        const int r = idx >> 2, q = idx & 3;
        float4 hi, lo;
        split4(load4(r, ch * TC_KC + 4 * q), hi, lo);
        sts128(s.a_hi + sw64(r, q), hi);
        sts128(s.a_lo + sw64(r, q), lo);
    }
    const int4* src = reinterpret_cast<const int4*>(img + (size_t)ch * 2 * N * 16);
    for (int idx = tid; idx < TcCfg<N>::B_BYTES / 16; idx += blockDim.x) {
        const int4 v = __ldg(src + idx);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(s.b + 16 * idx), "r"(v.x), "r"(v.y),
                     "r"(v.z), "r"(v.w) : "memory");
    }
}

template <int N>
__device__ __forceinline__ void issue_chunk(const StageLayout& s, uint32_t tmem, bool first) {
    constexpr uint32_t idesc = idesc_tf32(TC_BM, TcCfg<N>::MMA_N);
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
        const uint64_t ahi = sdesc(s.a_hi + 32 * kk, 512, kSW64);
        const uint64_t alo = sdesc(s.a_lo + 32 * kk, 512, kSW64);
#pragma unroll
        for (int nh = 0; nh < N / TcCfg<N>::MMA_N; ++nh) {
            const uint32_t boff = nh * TcCfg<N>::MMA_N * 64;
            const uint64_t bhi = sdesc(s.b + boff + 32 * kk, 512, kSW64);
            const uint64_t blo = sdesc(s.b + N * 64 + boff + 32 * kk, 512, kSW64);
            const uint32_t d = tmem + nh * TcCfg<N>::MMA_N;
            mma_tf32(d, ahi, bhi, idesc, (first && kk == 0) ? 0u : 1u);
            mma_tf32(d, ahi, blo, idesc, 1u);
            mma_tf32(d, alo, bhi, idesc, 1u);
        }
    }
}

// Runs the whole K loop; returns with the accumulator complete and visible.
template <int N, class LoadA>
__device__ __forceinline__ void tc_mainloop(uint8_t* smem_base, uint64_t* bars, uint32_t tmem, int nch,
                                            const float* __restrict__ img, LoadA load4) {
    using C = TcCfg<N>;
    const uint32_t base = smem_u32(smem_base);
    StageLayout st[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const uint32_t b0 = base + s * C::STAGE;
        st[s] = StageLayout{b0, b0 + C::A_BYTES, b0 + 2 * C::A_BYTES};
    }
    for (int ch = 0; ch < nch; ++ch) {
        const int s = ch & 1;
        if (ch >= 2) mbar_wait(&bars[s], ((ch - 2) >> 1) & 1);   // MMAs of chunk ch-2 released the stage
        stage_chunk<N>(st[s], ch, img, load4);
        fence_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_after();
            issue_chunk<N>(st[s], tmem, ch == 0);
            commit(&bars[s]);
        }
    }
    const int last = nch - 1;
    mbar_wait(&bars[last & 1], (last >> 1) & 1);
    fence_after();
}

template <int N>
__device__ __forceinline__ uint32_t tc_setup(uint8_t*& smem_base, uint64_t*& bars) {
    extern __shared__ uint8_t tc_smem_raw[];
    const uint32_t raw = smem_u32(tc_smem_raw);
    const uint32_t pad = (1024 - (raw & 1023)) & 1023;
    smem_base = tc_smem_raw + pad;
    bars = reinterpret_cast<uint64_t*>(smem_base + 2 * TcCfg<N>::STAGE);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
    if (threadIdx.x < 32) tmem_alloc(tslot, TcCfg<N>::TMEM_COLS);
    if (threadIdx.x == 32) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();
    return *tslot;
}

template <int N>
__device__ __forceinline__ void tc_teardown(uint32_t tmem) {
    fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, TcCfg<N>::TMEM_COLS);
}

// ---------------------------------------------------------------------------
// GEMM self-test entry: D[M x N] = A[M x K] B[N x K]^T (fp32 in/out)

template <int N>
__global__ void __launch_bounds__(256) tc_gemm_kernel(int M, int K, const float* __restrict__ a, int64_t lda,
                                                      const float* __restrict__ img, float* __restrict__ d,
                                                      int64_t ldd) {
    uint8_t* smem;
    uint64_t* bars;
    const uint32_t tmem = tc_setup<N>(smem, bars);
    const int64_t row0 = blockIdx.x * (int64_t)TC_BM;
    const int nch = (K + TC_KC - 1) / TC_KC;
    tc_mainloop<N>(smem, bars, tmem, nch, img, [&](int r, int k) {
        const int64_t g = row0 + r;
        if (g >= M || k >= K) return make_float4(0.f, 0.f, 0.f, 0.f);
        return *reinterpret_cast<const float4*>(a + g * lda + k);
    });
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, half = w >> 2;
    const int64_t row = row0 + 32 * q + lane;
    for (int c0 = half * 8; c0 < N; c0 += 16) {
        float v[8];
        tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + c0, v);
        tmem_wait_ld();
        if (row < M)
            for (int j = 0; j < 8; ++j) d[row * ldd + c0 + j] = v[j];
    }
    tc_teardown<N>(tmem);
}

// ---------------------------------------------------------------------------
// LSTM forward step on tcgen05

template <int HP>
__global__ void __launch_bounds__(256, (HP <= 64 ? 2 : 1)) lstm_fwd_tc_kernel(
    int64_t rows, int kx, const float* __restrict__ x, int64_t ldx, const float* __restrict__ hprev,
    const float* __restrict__ cprev, const float* __restrict__ img, const float* __restrict__ bias,
    float* __restrict__ hout, float* __restrict__ cout, float* __restrict__ gates) {
    constexpr int N = 4 * HP;
    uint8_t* smem;
    uint64_t* bars;
    const uint32_t tmem = tc_setup<N>(smem, bars);
    const int64_t row0 = blockIdx.x * (int64_t)TC_BM;
    const int K = kx + HP;
    const int nch = (K + TC_KC - 1) / TC_KC;
    tc_mainloop<N>(smem, bars, tmem, nch, img, [&](int r, int k) {
        const int64_t g = row0 + r;
        if (g >= rows || k >= K) return make_float4(0.f, 0.f, 0.f, 0.f);
        return k < kx ? __ldg(reinterpret_cast<const float4*>(x + g * ldx + k))
                      : __ldg(reinterpret_cast<const float4*>(hprev + g * HP + (k - kx)));
    });
    // epilogue: warp w reads TMEM lanes 32*(w&3).., units [half*HP/2, (half+1)*HP/2)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, half = w >> 2;
    const int64_t row = row0 + 32 * q + lane;
    const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
    for (int u0 = half * (HP / 2); u0 < (half + 1) * (HP / 2); u0 += 8) {
        float z[4][8];
#pragma unroll
        for (int g = 0; g < 4; ++g) tmem_ld8(tq + g * HP + u0, z[g]);
        tmem_wait_ld();
        if (row >= rows) continue;
        float cp[8], hv[8], cv[8], gi[8], gf[8], go[8], gg[8];
        *reinterpret_cast<float4*>(cp) = __ldg(reinterpret_cast<const float4*>(cprev + row * HP + u0));
        *reinterpret_cast<float4*>(cp + 4) = __ldg(reinterpret_cast<const float4*>(cprev + row * HP + u0 + 4));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            gi[j] = sigmoidf_acc(z[0][j] + __ldg(bias + 0 * HP + u0 + j));
            gf[j] = sigmoidf_acc(z[1][j] + __ldg(bias + 1 * HP + u0 + j));
            go[j] = sigmoidf_acc(z[2][j] + __ldg(bias + 2 * HP + u0 + j));
            gg[j] = tanhf(z[3][j] + __ldg(bias + 3 * HP + u0 + j));
            cv[j] = gf[j] * cp[j] + gi[j] * gg[j];
            hv[j] = go[j] * tanhf(cv[j]);
        }
        float4* ho = reinterpret_cast<float4*>(hout + row * HP + u0);
        float4* co = reinterpret_cast<float4*>(cout + row * HP + u0);
        ho[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
        ho[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
        co[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
        co[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
        if (gates) {
            float* gr = gates + row * N + u0;
            float* src[4] = {gi, gf, go, gg};
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                float4* o = reinterpret_cast<float4*>(gr + g * HP);
                o[0] = make_float4(src[g][0], src[g][1], src[g][2], src[g][3]);
                o[1] = make_float4(src[g][4], src[g][5], src[g][6], src[g][7]);
            }
        }
    }
    tc_teardown<N>(tmem);
}

template <int N>
int tc_gemm_t(int M, int K, const float* a, int64_t lda, const float* img, float* d, int64_t ldd, cudaStream_t st) {
    auto k = tc_gemm_kernel<N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<N>::SMEM);
    note_launch();
    k<<<(unsigned)cdiv(M, TC_BM), 256, TcCfg<N>::SMEM, st>>>(M, K, a, lda, img, d, ldd);
    return launch_status("tc_gemm_test");
}

template <int HP>
int lstm_fwd_tc_t(int64_t rows, int kx, const float* x, int64_t ldx, const float* hp_, const float* cp,
                  const float* img, const float* b, float* h, float* c, float* gates, cudaStream_t st) {
    constexpr int N = 4 * HP;
    auto k = lstm_fwd_tc_kernel<HP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<N>::SMEM);
    note_launch();
    k<<<(unsigned)cdiv(rows, TC_BM), 256, TcCfg<N>::SMEM, st>>>(rows, kx, x, ldx, hp_, cp, img, b, h, c, gates);
    return launch_status("lstm_forward_step_tc");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

size_t dgnn_tc_weight_image_bytes(int32_t n, int32_t k) {
    return (size_t)((k + TC_KC - 1) / TC_KC) * 2 * n * 64;
}

int dgnn_tc_weight_image(int32_t n, int32_t k, const float* w, int64_t ldw, float* img, void* stream) {
    DGNN_CHECK_ARG(n % 16 == 0 && n >= 16 && n <= 512 && k > 0, "tc_weight_image: n must be a multiple of 16 in [16, 512]");
    const int64_t total = (int64_t)((k + TC_KC - 1) / TC_KC) * n * 4;
    note_launch();
    wimg_kernel<<<(unsigned)cdiv(total, 256), 256, 0, as_stream(stream)>>>(n, k, w, ldw, img);
    return launch_status("tc_weight_image");
}

int dgnn_tc_gemm_test(int32_t m, int32_t n, int32_t k, const float* a, int64_t lda, const float* img, float* d,
                      int64_t ldd, void* stream) {
    DGNN_CHECK_ARG(k % 4 == 0 && lda % 4 == 0, "tc_gemm_test: k and lda must be multiples of 4");
    cudaStream_t st = as_stream(stream);
    switch (n) {
        case 64: return tc_gemm_t<64>(m, k, a, lda, img, d, ldd, st);
        case 128: return tc_gemm_t<128>(m, k, a, lda, img, d, ldd, st);
        case 256: return tc_gemm_t<256>(m, k, a, lda, img, d, ldd, st);
    }
    set_error("tc_gemm_test: n must be 64, 128 or 256");
    return DGNN_EUNSUPPORTED;
}

int dgnn_lstm_forward_step_tc(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                              const float* h_prev, const float* c_prev, const float* wimg, const float* bias,
                              float* h_out, float* c_out, float* gates, void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && kx % 4 == 0 && ldx % 4 == 0, "lstm_forward_step_tc: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 16: return lstm_fwd_tc_t<16>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
        case 32: return lstm_fwd_tc_t<32>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
        case 64: return lstm_fwd_tc_t<64>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
        case 128: return lstm_fwd_tc_t<128>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
    }
    set_error("lstm_forward_step_tc: unsupported hp %d", hp);
    return DGNN_EUNSUPPORTED;
}

}  // extern "C"
