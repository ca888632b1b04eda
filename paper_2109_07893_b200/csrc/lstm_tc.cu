// Temporal stage on the 5th-generation tensor cores (K5/K6).
//
// Forward step: z = [x | h_prev] W + b runs as tcgen05.mma kind::tf32 with
// the 3xTF32 split (fp32-accurate operands), accumulator in TMEM; the cell
// update (sigmoid/tanh, c = f c_prev + i g, h = o tanh c) is the epilogue,
// fed by tcgen05.ld, so z never touches HBM.  Reference training.py:370-391.
//
// Backward step: the gate-gradient pointwise (training.py:405-421) is the
// operand producer -- it computes dz for 4 hidden units per K chunk, writes dz
// (in place of the gate cache, for the weight-gradient GEMM) and dc, and
// stages dz as the A operand; [dx | dh] = dz W^T accumulates in TMEM and the
// epilogue streams it out.  The reduction dimension is taken unit-major
// (k = 4u + g) so one 16-wide chunk covers whole units; the weight image is
// permuted to match.
//
// Shared machinery: CTA = 128 rows (M = 128) x N columns (N = 4*HP forward,
// kx+HP rounded to 16 backward; N > 256 issues 256-wide slices).  K streams
// in chunks of 16 fp32 through a 2-stage shared-memory ring (SWIZZLE_64B
// K-major tiles): all threads stage the activation chunk (fp32 -> tf32 hi/lo)
// and copy the pre-split, pre-swizzled weight chunk; one thread issues the
// MMAs and commits them to the stage's mbarrier, so staging of chunk c+1
// overlaps the MMAs of chunk c.  <= 256 TMEM columns and 80-96 KB of smem
// per CTA give two CTAs per SM, overlapping one CTA's epilogue with the
// other's MMAs.
//
// Numerics: tcgen05 fp32 accumulation truncates (measured mean bias about
// -2.5e-8 relative per accumulate); with K <= 384 per step that stays
// ~1e-6 relative.  Long reductions must not accumulate in TMEM (see dW).
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

constexpr int TC_BM = 128;
constexpr int TC_KC = 16;  // fp32 K-elements per staged chunk (one SW64 row)
constexpr int TC_A_BYTES = TC_BM * 64;

__host__ __device__ inline int tmem_cols_for(int n) {
    return n <= 32 ? 32 : (n <= 64 ? 64 : (n <= 128 ? 128 : (n <= 256 ? 256 : 512)));
}
__host__ __device__ inline int tc_stage_bytes(int n) { return 2 * TC_A_BYTES + 2 * n * 64; }
inline size_t tc_smem_bytes(int n) { return (size_t)2 * tc_stage_bytes(n) + 1024 + 64; }

// Weight image for the B operand: [chunk][hi|lo][n_alloc rows][16 fp32], each
// [n_alloc][16] block an SW64 tile (byte-identical to its smem copy).  Row n
// (< n_valid) is row n of w (K-major, leading dimension ldw); with perm_hp > 0
// the K order is unit-major: element k reads w column (k % 4) * perm_hp + k / 4.
__global__ void wimg_kernel(int n_alloc, int n_valid, int K, const float* __restrict__ w, int64_t ldw,
                            int perm_hp, float* __restrict__ img) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int nch = (K + TC_KC - 1) / TC_KC;
    if (i >= (int64_t)nch * n_alloc * 4) return;
    const int q = (int)(i & 3);
    const int n = (int)((i >> 2) % n_alloc);
    const int ch = (int)(i / (4 * (int64_t)n_alloc));
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int k = ch * TC_KC + 4 * q + j;
        const int src = perm_hp > 0 ? (k % 4) * perm_hp + k / 4 : k;
        v[j] = (k < K && n < n_valid) ? w[(int64_t)n * ldw + src] : 0.f;
    }
    float4 hi, lo;
    split4(make_float4(v[0], v[1], v[2], v[3]), hi, lo);
    char* base = reinterpret_cast<char*>(img) + (size_t)ch * 2 * n_alloc * 64;
    *reinterpret_cast<float4*>(base + sw64(n, q)) = hi;
    *reinterpret_cast<float4*>(base + (size_t)n_alloc * 64 + sw64(n, q)) = lo;
}

// ---------------------------------------------------------------------------
// shared mainloop: D[128 x N] (TMEM) = A[128 x K] * B[N x K]^T, 3xTF32

struct Ring {
    uint32_t a_hi[2], a_lo[2], b[2];
    uint64_t* bars;   // [0..1] stage empty (MMA commit), [2..3] stage full (weight bulk copy)
    uint32_t tmem;
    int N;
};

__device__ __forceinline__ Ring tc_setup(int N) {
    extern __shared__ uint8_t tc_smem_raw[];
    const uint32_t raw = smem_u32(tc_smem_raw);
    const uint32_t pad = (1024 - (raw & 1023)) & 1023;
    uint8_t* base = tc_smem_raw + pad;
    Ring R;
    R.N = N;
    const int stage = tc_stage_bytes(N);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const uint32_t b0 = smem_u32(base) + s * stage;
        R.a_hi[s] = b0;
        R.a_lo[s] = b0 + TC_A_BYTES;
        R.b[s] = b0 + 2 * TC_A_BYTES;
    }
    R.bars = reinterpret_cast<uint64_t*>(base + 2 * stage);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(R.bars + 4);
    if (threadIdx.x < 32) tmem_alloc(tslot, tmem_cols_for(N));
    if (threadIdx.x == 32) {
#pragma unroll
        for (int i = 0; i < 4; ++i) mbar_init(&R.bars[i], 1);
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();
    R.tmem = *tslot;
    return R;
}

__device__ __forceinline__ void tc_teardown(const Ring& R) {
    fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(R.tmem, tmem_cols_for(R.N));
}

__device__ __forceinline__ void tc_issue(const Ring& R, int s, bool first) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
        const uint64_t ahi = sdesc(R.a_hi[s] + 32 * kk, 512, kSW64);
        const uint64_t alo = sdesc(R.a_lo[s] + 32 * kk, 512, kSW64);
        for (int n0 = 0; n0 < R.N; n0 += 256) {
            const int nn = R.N - n0 < 256 ? R.N - n0 : 256;
            const uint32_t idesc = idesc_tf32(TC_BM, nn);
            const uint64_t bhi = sdesc(R.b[s] + n0 * 64 + 32 * kk, 512, kSW64);
            const uint64_t blo = sdesc(R.b[s] + R.N * 64 + n0 * 64 + 32 * kk, 512, kSW64);
            const uint32_t d = R.tmem + n0;
            mma_tf32(d, ahi, bhi, idesc, (first && kk == 0) ? 0u : 1u);
            mma_tf32(d, ahi, blo, idesc, 1u);
            mma_tf32(d, alo, bhi, idesc, 1u);
        }
    }
}

// The A operand is produced in two steps so global latency overlaps the
// previous chunk: `fetch(ch, item)` issues the loads for one item (row
// item / 4, 16-byte column group item % 4 of chunk ch) into a register
// payload one chunk ahead; `produce(payload, ch, item)` turns it into the 4
// fp32 values to stage (it runs exactly once per item, so it may have side
// effects).  The weight chunk arrives by one cp.async.bulk on the stage's
// "full" barrier.  Requires blockDim.x == 256.
template <class Fetch, class Produce>
__device__ __forceinline__ void tc_mainloop(const Ring& R, int nch, const float* __restrict__ img, Fetch fetch,
                                            Produce produce) {
    constexpr int ITEMS = TC_BM * 4 / 256;
    using Payload = decltype(fetch(0, 0));
    const int tid = threadIdx.x;
    const uint32_t b_bytes = (uint32_t)(2 * R.N * 64);
    const char* img_bytes = reinterpret_cast<const char*>(img);
    uint64_t* empty = R.bars;
    uint64_t* full = R.bars + 2;
    Payload cur[ITEMS], nxt[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) cur[i] = fetch(0, tid + 256 * i);
    for (int ch = 0; ch < nch; ++ch) {
        const int s = ch & 1;
        if (ch + 1 < nch) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) nxt[i] = fetch(ch + 1, tid + 256 * i);
        }
        if (ch >= 2) mbar_wait(&empty[s], ((ch - 2) >> 1) & 1);   // MMAs of chunk ch-2 released the stage
        if (tid == 0) {
            mbar_arrive_expect_tx(&full[s], b_bytes);
            bulk_g2s(R.b[s], img_bytes + (size_t)ch * b_bytes, b_bytes, &full[s]);
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int idx = tid + 256 * i;
            const int r = idx >> 2, q = idx & 3;
            float4 hi, lo;
            split4(produce(cur[i], ch, idx), hi, lo);
            sts128(R.a_hi[s] + sw64(r, q), hi);
            sts128(R.a_lo[s] + sw64(r, q), lo);
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            mbar_wait(&full[s], (ch >> 1) & 1);
            fence_after();
            tc_issue(R, s, ch == 0);
            commit(&empty[s]);
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) cur[i] = nxt[i];
    }
    const int last = nch - 1;
    mbar_wait(&empty[last & 1], (last >> 1) & 1);
    fence_after();
}

struct Raw4 {
    float4 v;
};

__device__ __forceinline__ float4 pass4(const Raw4& p, int, int) { return p.v; }

// ---------------------------------------------------------------------------
// GEMM self-test entry: D[M x N] = A[M x K] B[N x K]^T (fp32 in/out)

__global__ void __launch_bounds__(256) tc_gemm_kernel(int M, int N, int K, const float* __restrict__ a, int64_t lda,
                                                      const float* __restrict__ img, float* __restrict__ d,
                                                      int64_t ldd) {
    const Ring R = tc_setup(N);
    const int64_t row0 = blockIdx.x * (int64_t)TC_BM;
    const int nch = (K + TC_KC - 1) / TC_KC;
    tc_mainloop(
        R, nch, img,
        [&](int ch, int idx) {
            const int64_t g = row0 + (idx >> 2);
            const int k = ch * TC_KC + 4 * (idx & 3);
            Raw4 p{make_float4(0.f, 0.f, 0.f, 0.f)};
            if (g < M && k < K) p.v = __ldg(reinterpret_cast<const float4*>(a + g * lda + k));
            return p;
        },
        pass4);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, half = w >> 2;
    const int64_t row = row0 + 32 * q + lane;
    for (int c0 = half * 8; c0 < N; c0 += 16) {
        float v[8];
        tmem_ld8(R.tmem + ((uint32_t)(32 * q) << 16) + c0, v);
        tmem_wait_ld();
        if (row < M)
            for (int j = 0; j < 8; ++j) d[row * ldd + c0 + j] = v[j];
    }
    tc_teardown(R);
}

// ---------------------------------------------------------------------------
// LSTM forward step

template <int HP>
__global__ void __launch_bounds__(256, (HP <= 64 ? 2 : 1)) lstm_fwd_tc_kernel(
    int64_t rows, int kx, const float* __restrict__ x, int64_t ldx, const float* __restrict__ hprev,
    const float* __restrict__ cprev, const float* __restrict__ img, const float* __restrict__ bias,
    float* __restrict__ hout, float* __restrict__ cout, float* __restrict__ gates) {
    constexpr int N = 4 * HP;
    const Ring R = tc_setup(N);
    const int64_t row0 = blockIdx.x * (int64_t)TC_BM;
    const int K = kx + HP;
    const int nch = (K + TC_KC - 1) / TC_KC;
    tc_mainloop(
        R, nch, img,
        [&](int ch, int idx) {
            const int64_t g = row0 + (idx >> 2);
            const int k = ch * TC_KC + 4 * (idx & 3);
            Raw4 p{make_float4(0.f, 0.f, 0.f, 0.f)};
            if (g < rows && k < K)
                p.v = k < kx ? __ldg(reinterpret_cast<const float4*>(x + g * ldx + k))
                             : __ldg(reinterpret_cast<const float4*>(hprev + g * HP + (k - kx)));
            return p;
        },
        pass4);
    // epilogue: warp w reads TMEM lanes 32*(w&3).., units [half*HP/2, (half+1)*HP/2)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, half = w >> 2;
    const int64_t row = row0 + 32 * q + lane;
    const uint32_t tq = R.tmem + ((uint32_t)(32 * q) << 16);
    for (int u0 = half * (HP / 2); u0 < (half + 1) * (HP / 2); u0 += 8) {
        float z[4][8];
#pragma unroll
        for (int g = 0; g < 4; ++g) tmem_ld8(tq + g * HP + u0, z[g]);
        tmem_wait_ld();
        if (row >= rows) continue;
        float cp[8], hv[8], cv[8], gi[8], gf[8], go[8], gg[8];
        *reinterpret_cast<float4*>(cp) = __ldg(reinterpret_cast<const float4*>(cprev + tb_off(row, u0, HP, rows)));
        *reinterpret_cast<float4*>(cp + 4) =
            __ldg(reinterpret_cast<const float4*>(cprev + tb_off(row, u0 + 4, HP, rows)));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            gi[j] = act_sigmoid(z[0][j] + __ldg(bias + 0 * HP + u0 + j));
            gf[j] = act_sigmoid(z[1][j] + __ldg(bias + 1 * HP + u0 + j));
            go[j] = act_sigmoid(z[2][j] + __ldg(bias + 2 * HP + u0 + j));
            gg[j] = act_tanh(z[3][j] + __ldg(bias + 3 * HP + u0 + j));
            cv[j] = gf[j] * cp[j] + gi[j] * gg[j];
            hv[j] = go[j] * act_tanh(cv[j]);
        }
        float4* ho = reinterpret_cast<float4*>(hout + row * HP + u0);
        ho[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
        ho[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
        *reinterpret_cast<float4*>(cout + tb_off(row, u0, HP, rows)) = make_float4(cv[0], cv[1], cv[2], cv[3]);
        *reinterpret_cast<float4*>(cout + tb_off(row, u0 + 4, HP, rows)) = make_float4(cv[4], cv[5], cv[6], cv[7]);
        if (gates) {
            float* src[4] = {gi, gf, go, gg};
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                *reinterpret_cast<float4*>(gates + tb_off(row, g * HP + u0, N, rows)) =
                    make_float4(src[g][0], src[g][1], src[g][2], src[g][3]);
                *reinterpret_cast<float4*>(gates + tb_off(row, g * HP + u0 + 4, N, rows)) =
                    make_float4(src[g][4], src[g][5], src[g][6], src[g][7]);
            }
        }
    }
    tc_teardown(R);
}

// ---------------------------------------------------------------------------
// LSTM backward step

template <int HP>
__global__ void __launch_bounds__(256, 2) lstm_bwd_tc_kernel(
    int64_t rows, int kx, int N, const float* __restrict__ dy, const float* __restrict__ dh_in,
    const float* __restrict__ dc_in, float* gates, const float* __restrict__ cprev, const float* __restrict__ cnew,
    const float* __restrict__ img, float* __restrict__ dx, int64_t lddx, float* __restrict__ dh_out,
    float* __restrict__ dc_out) {
    constexpr int NC = 4 * HP;
    const Ring R = tc_setup(N);
    const int64_t row0 = blockIdx.x * (int64_t)TC_BM;
    // K chunk ch covers units 4ch..4ch+3; column k = 4u + g
    struct Cell {
        float gi, gf, go, gg, cp, cn, dh, dc;
    };
    tc_mainloop(
        R, HP / 4, img,
        [&](int ch, int idx) {
            const int64_t g = row0 + (idx >> 2);
            const int u = 4 * ch + (idx & 3);
            Cell p{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (g < rows) {
                const int64_t o = g * HP + u, ob = tb_off(g, u, HP, rows);
                p.gi = gates[tb_off(g, u, NC, rows)];
                p.gf = gates[tb_off(g, HP + u, NC, rows)];
                p.go = gates[tb_off(g, 2 * HP + u, NC, rows)];
                p.gg = gates[tb_off(g, 3 * HP + u, NC, rows)];
                p.cp = __ldg(cprev + ob);
                p.cn = __ldg(cnew + ob);
                p.dh = (dy ? __ldg(dy + o) : 0.f) + __ldg(dh_in + o);
                p.dc = __ldg(dc_in + ob);
            }
            return p;
        },
        [&](const Cell& p, int ch, int idx) {
            const int64_t g = row0 + (idx >> 2);
            if (g >= rows) return make_float4(0.f, 0.f, 0.f, 0.f);
            const int u = 4 * ch + (idx & 3);
            const float tcn = act_tanh(p.cn);
            const float d_o = p.dh * tcn;
            const float dc = p.dh * p.go * (1.f - tcn * tcn) + p.dc;
            const float df = dc * p.cp, di = dc * p.gg, dg = dc * p.gi;
            dc_out[tb_off(g, u, HP, rows)] = dc * p.gf;
            const float z0 = di * p.gi * (1.f - p.gi);
            const float z1 = df * p.gf * (1.f - p.gf);
            const float z2 = d_o * p.go * (1.f - p.go);
            const float z3 = dg * (1.f - p.gg * p.gg);
            // dz replaces the gate cache (training.py:413-421)
            gates[tb_off(g, u, NC, rows)] = z0;
            gates[tb_off(g, HP + u, NC, rows)] = z1;
            gates[tb_off(g, 2 * HP + u, NC, rows)] = z2;
            gates[tb_off(g, 3 * HP + u, NC, rows)] = z3;
            return make_float4(z0, z1, z2, z3);
        });
    const int K = kx + HP;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, q = w & 3, half = w >> 2;
    const int64_t row = row0 + 32 * q + lane;
    const uint32_t tq = R.tmem + ((uint32_t)(32 * q) << 16);
    for (int c0 = half * 8; c0 < N; c0 += 16) {
        float v[8];
        tmem_ld8(tq + c0, v);
        tmem_wait_ld();
        if (row >= rows) continue;
#pragma unroll
        for (int h4 = 0; h4 < 2; ++h4) {
            const int c = c0 + 4 * h4;
            const float4 val = make_float4(v[4 * h4], v[4 * h4 + 1], v[4 * h4 + 2], v[4 * h4 + 3]);
            if (c < kx) *reinterpret_cast<float4*>(dx + row * lddx + c) = val;
            else if (c < K) *reinterpret_cast<float4*>(dh_out + row * HP + (c - kx)) = val;
        }
    }
    tc_teardown(R);
}

template <class Kern>
static void set_smem(Kern k, size_t bytes) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int HP>
int lstm_fwd_tc_t(int64_t rows, int kx, const float* x, int64_t ldx, const float* hp_, const float* cp,
                  const float* img, const float* b, float* h, float* c, float* gates, cudaStream_t st) {
    auto k = lstm_fwd_tc_kernel<HP>;
    const size_t smem = tc_smem_bytes(4 * HP);
    set_smem(k, smem);
    note_launch();
    k<<<(unsigned)cdiv(rows, TC_BM), 256, smem, st>>>(rows, kx, x, ldx, hp_, cp, img, b, h, c, gates);
    return launch_status("lstm_forward_step_tc");
}

template <int HP>
int lstm_bwd_tc_t(int64_t rows, int kx, const float* dy, const float* dh_in, const float* dc_in, float* gates,
                  const float* cp, const float* cn, const float* img, float* dx, int64_t lddx, float* dh_out,
                  float* dc_out, cudaStream_t st) {
    const int N = (kx + HP + 15) / 16 * 16;
    if (N > 256) {
        set_error("lstm_backward_step_tc: kx + hp = %d exceeds 256", kx + HP);
        return DGNN_EUNSUPPORTED;
    }
    auto k = lstm_bwd_tc_kernel<HP>;
    const size_t smem = tc_smem_bytes(N);
    set_smem(k, smem);
    note_launch();
    k<<<(unsigned)cdiv(rows, TC_BM), 256, smem, st>>>(rows, kx, N, dy, dh_in, dc_in, gates, cp, cn, img, dx, lddx,
                                                        dh_out, dc_out);
    return launch_status("lstm_backward_step_tc");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

size_t dgnn_tc_weight_image_bytes(int32_t n, int32_t k) {
    return (size_t)((k + TC_KC - 1) / TC_KC) * 2 * n * 64;
}

int dgnn_tc_weight_image_ex(int32_t n_alloc, int32_t n_valid, int32_t k, const float* w, int64_t ldw,
                            int32_t perm_hp, float* img, void* stream) {
    DGNN_CHECK_ARG(n_alloc % 16 == 0 && n_alloc >= 16 && n_alloc <= 512 && n_valid <= n_alloc && k > 0,
                   "tc_weight_image: n_alloc must be a multiple of 16 in [16, 512]");
    const int64_t total = (int64_t)((k + TC_KC - 1) / TC_KC) * n_alloc * 4;
    note_launch();
    wimg_kernel<<<(unsigned)cdiv(total, 256), 256, 0, as_stream(stream)>>>(n_alloc, n_valid, k, w, ldw, perm_hp, img);
    return launch_status("tc_weight_image");
}

int dgnn_tc_weight_image(int32_t n, int32_t k, const float* w, int64_t ldw, float* img, void* stream) {
    return dgnn_tc_weight_image_ex(n, n, k, w, ldw, 0, img, stream);
}

int dgnn_tc_gemm_test(int32_t m, int32_t n, int32_t k, const float* a, int64_t lda, const float* img, float* d,
                      int64_t ldd, void* stream) {
    DGNN_CHECK_ARG(k % 4 == 0 && lda % 4 == 0 && n % 16 == 0 && n >= 16 && n <= 512,
                   "tc_gemm_test: k, lda multiples of 4; n a multiple of 16 in [16, 512]");
    cudaStream_t st = as_stream(stream);
    const size_t smem = tc_smem_bytes(n);
    set_smem(tc_gemm_kernel, smem);
    note_launch();
    tc_gemm_kernel<<<(unsigned)cdiv(m, TC_BM), 256, smem, st>>>(m, n, k, a, lda, img, d, ldd);
    return launch_status("tc_gemm_test");
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

int dgnn_lstm_backward_step_tc(int64_t rows, int32_t kx, int32_t hp, const float* dy, const float* dh_in,
                               const float* dc_in, float* gates, const float* c_prev, const float* c_new,
                               const float* wimg, float* dx, int64_t lddx, float* dh_out, float* dc_out,
                               void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && kx % 4 == 0 && lddx % 4 == 0, "lstm_backward_step_tc: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 16: return lstm_bwd_tc_t<16>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wimg, dx, lddx, dh_out, dc_out, st);
        case 32: return lstm_bwd_tc_t<32>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wimg, dx, lddx, dh_out, dc_out, st);
        case 64: return lstm_bwd_tc_t<64>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wimg, dx, lddx, dh_out, dc_out, st);
    }
    set_error("lstm_backward_step_tc: unsupported hp %d (use the SIMT step)", hp);
    return DGNN_EUNSUPPORTED;
}

}  // extern "C"
