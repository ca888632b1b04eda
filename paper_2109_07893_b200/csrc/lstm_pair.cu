// K5 on CTA pairs: the LSTM forward step with tcgen05.mma.cta_group::2.
//
// Why: the warp-specialised one-CTA kernel (lstm_ws.cu) streams the whole
// 3xTF32 weight image (2 x (F_in + H) x 4H fp32, 384 KB at hidden 64) from L2
// into shared memory for every 128-row tile -- 4x the activation bytes of
// the tile.  At the MMA pace that is ~6 KB/cycle of L2->SM traffic across
// the chip, the whole L2 read path (B300_MICROARCH: ~6300 B/cyc), so the
// tensor pipe starves.  A CTA pair (two SMs of one TPC, a 2-CTA cluster)
// runs one M = 256 MMA per K step: each CTA stages its own 128 rows of the
// activations and only HALF of the weight chunk (N/2 gate columns); the
// tensor cores of the pair read the other half from the peer's shared
// memory.  Weight traffic per row halves, and the smaller stage (32 KB
// instead of 48 KB at hidden 64) deepens the ring from 4 to 6 stages.
//
// Roles per CTA (both CTAs):
//   warps 0..3  producers: cp.async this CTA's activation chunk LA chunks
//               ahead, split fp32 -> tf32 hi/lo in place, arrive full_a[s];
//               producer 0 bulk-copies this CTA's weight half (full_b[s]).
//   warp 4      leader CTA: the MMA issuer (one lane) waits for its own
//               stage and the peer's (peer_full[s], arrived remotely by the
//               peer's relay), issues the pair MMAs, commits empty[s] and
//               accfull[a] to BOTH CTAs (multicast commit).  Peer CTA: the
//               relay -- waits its own full_a/full_b and arrives on the
//               leader's peer_full[s].
//   warps 5..   epilogue: wait accfull[a], tcgen05.ld this CTA's 128 rows,
//               cell update, stores; arrive on the LEADER's accempty[a]
//               (2 x NEPI arrivals per phase).
// Same operand layouts (SW64 K-major), same 3xTF32 product order per K step
// and the same epilogue as lstm_ws.cu, so the results are bitwise equal.
// Reference: training.py:370-391.
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

namespace pairk {
constexpr int BM = 128;            // rows per CTA (the pair covers 256)
constexpr int KC = 16;             // K per chunk (two kind::tf32 K steps)
constexpr int A_TILE = BM * 64;    // one SW64 K-major tile of BM rows
constexpr int MAX_STAGES = 8;
constexpr int RING_BYTES = 192 * 1024;
// Bottleneck probe (scripts/pair_probe.cu builds with -DDGNN_PAIR_PROBE=mask):
// 1 no MMAs, 2 no activation loads (zeros), 4 no weight copies, 8 epilogue
// without cell math / stores, 16 without stores.  Always 0 in the library.
#ifndef DGNN_PAIR_PROBE
#define DGNN_PAIR_PROBE 0
#endif
constexpr int PROBE = DGNN_PAIR_PROBE;
}  // namespace pairk

template <int HP>
struct PairCfg {
    static constexpr int N = 4 * HP;                       // gate columns of the MMA
    static constexpr int NB = N / 2;                       // weight rows this CTA stages
    static constexpr int STAGE = 2 * pairk::A_TILE + 2 * NB * 64;
    static constexpr int RAW_STAGES = 8;                   // fp32 activation landing ring
    static constexpr int OP_BYTES = pairk::RING_BYTES - RAW_STAGES * pairk::A_TILE;
    static constexpr int STAGES = OP_BYTES / STAGE > pairk::MAX_STAGES ? pairk::MAX_STAGES : OP_BYTES / STAGE;
    static constexpr int NPROD = 8;
    static constexpr int MMA_WARP = 8;
    static constexpr int NEPI = HP >= 32 ? 16 : 8;
    static constexpr int THREADS = 32 * (NPROD + 1 + NEPI);
    static constexpr int NPT = 32 * NPROD;
    static constexpr int TMEM_COLS = 2 * N <= 32 ? 32 : (2 * N <= 64 ? 64 : (2 * N <= 128 ? 128 : (2 * N <= 256 ? 256 : 512)));
};

struct PairBars {
    uint64_t full_a[pairk::MAX_STAGES], full_b[pairk::MAX_STAGES], peer_full[pairk::MAX_STAGES],
        empty[pairk::MAX_STAGES], accfull[2], accempty[2];
    uint32_t tmem;
};

template <int HP>
__global__ void __launch_bounds__(PairCfg<HP>::THREADS, 1) lstm_fwd_pair_kernel(
    int64_t rows, int kx, const float* __restrict__ x, int64_t ldx, const float* __restrict__ hprev,
    const float* __restrict__ cprev, const float* __restrict__ img, const float* __restrict__ bias,
    float* __restrict__ hout, float* __restrict__ cout, float* __restrict__ gates) {
    using C = PairCfg<HP>;
    constexpr int N = C::N, NB = C::NB, S = C::STAGES;
    constexpr int ITEMS = pairk::BM * 4 / C::NPT;   // 2
    extern __shared__ uint8_t pair_smem_raw[];
    const uint32_t raw = smem_u32(pair_smem_raw);
    const uint32_t pad = (1024 - (raw & 1023)) & 1023;
    const uint32_t base = raw + pad;
    PairBars* bars = reinterpret_cast<PairBars*>(pair_smem_raw + pad + S * C::STAGE + C::RAW_STAGES * pairk::A_TILE);
    const uint32_t raw0 = base + S * C::STAGE;
    auto a_hi = [&](int s) { return base + s * C::STAGE; };
    auto a_lo = [&](int s) { return base + s * C::STAGE + pairk::A_TILE; };
    auto b_hi = [&](int s) { return base + s * C::STAGE + 2 * pairk::A_TILE; };
    auto b_lo = [&](int s) { return base + s * C::STAGE + 2 * pairk::A_TILE + NB * 64; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nst = (int)cdiv(rows, 2 * pairk::BM);
    const int K = kx + HP;
    const int nch = (K + pairk::KC - 1) / pairk::KC;
    const uint32_t b_bytes = 2 * N * 64;     // one chunk of the weight image (hi + lo, all N rows)
    const uint32_t half = NB * 64;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&bars->full_a[s], C::NPROD);
            mbar_init(&bars->full_b[s], 1);
            mbar_init(&bars->peer_full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->accfull[a], 1);
            mbar_init(&bars->accempty[a], 2 * C::NEPI);
        }
        fence_mbar_init();
    }
    if (warp == C::MMA_WARP) tmem_alloc2(&bars->tmem, C::TMEM_COLS);
    fence_before();
    __syncthreads();
    cluster_sync();          // both CTAs' barriers and TMEM exist before any remote arrive / pair MMA
    fence_after();

    const int my_st = pair < nst ? (int)cdiv(nst - pair, npairs) : 0;
    const uint32_t G = (uint32_t)my_st * nch;

    if (warp < C::NPROD) {
        // Activations land (cp.async, fp32) in a raw ring RS chunks deep,
        // decoupled from the operand ring: up to RS - 1 chunks (56 KB per
        // SM at RS = 8) are in flight, enough to cover HBM latency at the
        // MMA pace, while the operand stages stay few.  Each producer thread
        // loads, splits and reloads only its own items, so a raw slot needs
        // no barrier.
        constexpr int RS = C::RAW_STAGES;
        const int ptid = threadIdx.x;
        // the activation rows of a tile are contiguous in HBM but the chunks
        // read them 64 B at a time, 8..12 visits per row spread over the
        // tile: pull the next tile's whole blocks (x, h_prev, c_prev) into L2
        // with bulk prefetches first, so DRAM streams them sequentially
        auto prefetch_tile = [&](int st) {
            const int64_t t0 = (int64_t)st * 2 * pairk::BM + rank * pairk::BM;
            if (pairk::PROBE & 2 || t0 >= rows) return;
            const int64_t nr = rows - t0 < pairk::BM ? rows - t0 : pairk::BM;
            bulk_prefetch_l2(x + t0 * ldx, (uint32_t)(nr * ldx * 4));
            bulk_prefetch_l2(hprev + t0 * HP, (uint32_t)(nr * HP * 4));
            bulk_prefetch_l2(cprev + t0 * HP, (uint32_t)(nr * HP * 4));   // tile-blocked: one block
        };
        auto issue = [&](uint32_t g) {
            const int st = pair + (int)(g / nch) * npairs;
            const int ch = (int)(g % nch);
            if (ptid == 0 && ch == 0 && st + npairs < nst) prefetch_tile(st + npairs);
            const uint32_t slot = raw0 + (g % RS) * pairk::A_TILE;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int idx = ptid + C::NPT * i;
                const int r = idx >> 2, q = idx & 3;
                const int64_t gr = (int64_t)st * 2 * pairk::BM + rank * pairk::BM + r;
                const int k = ch * pairk::KC + 4 * q;
                const bool ok = gr < rows && k < K && !(pairk::PROBE & 2);
                const float* src = !ok ? x : (k < kx ? x + gr * ldx + k : hprev + gr * HP + (k - kx));
                cp_async16(slot + sw64(r, q), src, ok ? 16u : 0u);
            }
        };
        if (ptid == 0 && G) prefetch_tile(pair);
        for (uint32_t g = 0; g < (uint32_t)(RS - 1); ++g) {
            if (g < G) issue(g);
            cp_async_commit();
        }
        for (uint32_t g = 0; g < G; ++g) {
            const int s = g % S;
            const uint32_t j = g / S;
            if (j >= 1) mbar_wait(&bars->empty[s], (j - 1) & 1);
            if (ptid == 0 && (pairk::PROBE & 4)) {
                mbar_arrive(&bars->full_b[s]);
            } else if (ptid == 0) {
                const int ch = (int)(g % nch);
                mbar_arrive_expect_tx(&bars->full_b[s], 2 * half);
                const char* src = reinterpret_cast<const char*>(img) + (size_t)ch * b_bytes + rank * half;
                bulk_g2s(b_hi(s), src, half, &bars->full_b[s]);
                bulk_g2s(b_lo(s), src + N * 64, half, &bars->full_b[s]);
            }
            cp_async_wait<RS - 2>();
            const uint32_t slot = raw0 + (g % RS) * pairk::A_TILE;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int idx = ptid + C::NPT * i;
                const uint32_t off = sw64(idx >> 2, idx & 3);
                float4 hi, lo;
                split4(lds128(slot + off), hi, lo);
                sts128(a_hi(s) + off, hi);
                sts128(a_lo(s) + off, lo);
            }
            fence_async_smem();
            __syncwarp();
            if ((ptid & 31) == 0) mbar_arrive(&bars->full_a[s]);
            if (g + RS - 1 < G) issue(g + RS - 1);
            cp_async_commit();
        }
    } else if (warp == C::MMA_WARP) {
        if (lane == 0) {
            if (rank == 0) {
                const uint32_t idesc = idesc_tf32(2 * pairk::BM, N);
                uint32_t gc = 0;
                for (int it = 0; it < my_st; ++it) {
                    const uint32_t a = it & 1, u = it >> 1;
                    if (u >= 1) mbar_wait(&bars->accempty[a], (u - 1) & 1);
                    fence_after();
                    const uint32_t d = bars->tmem + a * N;
                    for (int ch = 0; ch < nch; ++ch, ++gc) {
                        const int s = gc % S;
                        const uint32_t j = gc / S;
                        mbar_wait(&bars->full_a[s], j & 1);
                        mbar_wait(&bars->full_b[s], j & 1);
                        mbar_wait(&bars->peer_full[s], j & 1);
                        fence_after();
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk) {
                            const uint64_t ahi = sdesc(a_hi(s) + 32 * kk, 512, kSW64);
                            const uint64_t alo = sdesc(a_lo(s) + 32 * kk, 512, kSW64);
                            const uint64_t bhi = sdesc(b_hi(s) + 32 * kk, 512, kSW64);
                            const uint64_t blo = sdesc(b_lo(s) + 32 * kk, 512, kSW64);
                            if (pairk::PROBE & 1) continue;
                            mma2_tf32(d, ahi, bhi, idesc, (ch == 0 && kk == 0) ? 0u : 1u);
                            mma2_tf32(d, ahi, blo, idesc, 1u);
                            mma2_tf32(d, alo, bhi, idesc, 1u);
                        }
                        commit2_mc(&bars->empty[s], 0x3);
                    }
                    commit2_mc(&bars->accfull[a], 0x3);
                }
            } else {
                // relay: this CTA's stage s is loaded -> tell the leader
                for (uint32_t g = 0; g < G; ++g) {
                    const int s = g % S;
                    const uint32_t j = g / S;
                    mbar_wait(&bars->full_a[s], j & 1);
                    mbar_wait(&bars->full_b[s], j & 1);
                    mbar_arrive_cta(&bars->peer_full[s], 0);
                }
            }
        }
        __syncwarp();
    } else {
        const int e = warp - C::MMA_WARP - 1;
        constexpr int UPW = HP / (C::NEPI / 4);   // units per epilogue warp
        const int q = warp & 3, part = e >> 2;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        for (int it = 0; it < my_st; ++it) {
            const int st = pair + it * npairs;
            const uint32_t a = it & 1, u = it >> 1;
            const int64_t row = (int64_t)st * 2 * pairk::BM + rank * pairk::BM + 32 * q + lane;
            const bool valid = row < rows;
            float cp[UPW];
#pragma unroll
            for (int i = 0; i < UPW / 4; ++i) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (valid) v = __ldg(reinterpret_cast<const float4*>(cprev + tb_off(row, part * UPW + 4 * i, HP, rows)));
                cp[4 * i] = v.x;
                cp[4 * i + 1] = v.y;
                cp[4 * i + 2] = v.z;
                cp[4 * i + 3] = v.w;
            }
            mbar_wait(&bars->accfull[a], u & 1);
            fence_after();
            const uint32_t tq = bars->tmem + lane_off + a * N;
#pragma unroll
            for (int g8 = 0; g8 < UPW / 8; ++g8) {
                const int u0 = part * UPW + 8 * g8;
                float z[4][8];
#pragma unroll
                for (int g = 0; g < 4; ++g) tmem_ld8(tq + g * HP + u0, z[g]);
                tmem_wait_ld();
                if (!valid || (pairk::PROBE & 8)) continue;
                float hv[8], cv[8], gi[8], gf[8], go[8], gg[8];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    gi[jj] = act_sigmoid(z[0][jj] + __ldg(bias + 0 * HP + u0 + jj));
                    gf[jj] = act_sigmoid(z[1][jj] + __ldg(bias + 1 * HP + u0 + jj));
                    go[jj] = act_sigmoid(z[2][jj] + __ldg(bias + 2 * HP + u0 + jj));
                    gg[jj] = act_tanh(z[3][jj] + __ldg(bias + 3 * HP + u0 + jj));
                    cv[jj] = gf[jj] * cp[8 * g8 + jj] + gi[jj] * gg[jj];
                    hv[jj] = go[jj] * act_tanh(cv[jj]);
                }
                if (pairk::PROBE & 16) {
                    float acc = 0.f;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) acc += hv[jj] + cv[jj] + gi[jj] + gf[jj] + go[jj] + gg[jj];
                    if (acc == 12345.f) hout[row] = acc;
                    continue;
                }
                float4* ho = reinterpret_cast<float4*>(hout + row * HP + u0);
                ho[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
                ho[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
                *reinterpret_cast<float4*>(cout + tb_off(row, u0, HP, rows)) = make_float4(cv[0], cv[1], cv[2], cv[3]);
                *reinterpret_cast<float4*>(cout + tb_off(row, u0 + 4, HP, rows)) =
                    make_float4(cv[4], cv[5], cv[6], cv[7]);
                if (gates) {
                    const float* src[4] = {gi, gf, go, gg};
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        *reinterpret_cast<float4*>(gates + tb_off(row, g * HP + u0, N, rows)) =
                            make_float4(src[g][0], src[g][1], src[g][2], src[g][3]);
                        *reinterpret_cast<float4*>(gates + tb_off(row, g * HP + u0 + 4, N, rows)) =
                            make_float4(src[g][4], src[g][5], src[g][6], src[g][7]);
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) mbar_arrive(&bars->accempty[a]);
                else mbar_arrive_cta(&bars->accempty[a], 0);
            }
        }
    }
    fence_before();
    __syncthreads();
    cluster_sync();          // the peer is done with every pair MMA / TMEM access
    if (warp == C::MMA_WARP) tmem_dealloc2(bars->tmem, C::TMEM_COLS);
}

template <int HP>
int lstm_fwd_pair_t(int64_t rows, int kx, const float* x, int64_t ldx, const float* hp_, const float* cp,
                    const float* img, const float* b, float* h, float* c, float* gates, cudaStream_t st) {
    using C = PairCfg<HP>;
    auto k = lstm_fwd_pair_kernel<HP>;
    const size_t smem = (size_t)C::STAGES * C::STAGE + (size_t)C::RAW_STAGES * pairk::A_TILE + 1024 +
                        sizeof(PairBars) + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int nst = (int)cdiv(rows, 2 * pairk::BM);
    int npairs = persistent_ctas() / 2;
    if (npairs > nst) npairs = nst;
    if (npairs < 1) npairs = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * npairs);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    note_launch();
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, rows, kx, x, ldx, hp_, cp, img, b, h, c, gates);
    if (e != cudaSuccess) {
        set_error("lstm_forward_step_pair: %s", cudaGetErrorString(e));
        return DGNN_ECUDA;
    }
    return launch_status("lstm_forward_step_pair");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

int dgnn_lstm_forward_step_pair(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                                const float* h_prev, const float* c_prev, const float* wimg, const float* bias,
                                float* h_out, float* c_out, float* gates, void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && kx % 4 == 0 && ldx % 4 == 0, "lstm_forward_step_pair: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 32: return lstm_fwd_pair_t<32>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
        case 64: return lstm_fwd_pair_t<64>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
    }
    set_error("lstm_forward_step_pair: unsupported hp %d (use dgnn_lstm_forward_step_ws)", hp);
    return DGNN_EUNSUPPORTED;
}

}  // extern "C"
