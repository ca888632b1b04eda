// Persistent, warp-specialised tcgen05 LSTM step kernels (K5 forward, K6
// backward).  Same math and operand conventions as lstm_tc.cu (3xTF32,
// SW64 K-major tiles, pre-split weight images), restructured so that HBM
// traffic, tensor-core work and the cell epilogue overlap:
//
//   warps 0..3  producers: fetch the activation chunk one chunk ahead,
//               split fp32 -> tf32 hi/lo, store the SW64 tile, arrive on
//               full_a[s]; producer 0 lane 0 also bulk-copies the weight
//               chunk (cp.async.bulk, complete_tx on full_b[s]).
//   warp 4      MMA issuer (one lane): waits full_a/full_b, issues the
//               3xTF32 MMAs into TMEM accumulator a (two buffers), commits
//               empty[s] per chunk and accfull[a] per tile.
//   warps 5..12 epilogue: wait accfull[a], tcgen05.ld, cell update (forward)
//               or dx/dh stores (backward), arrive accempty[a].
//
// One CTA per SM loops over 128-row tiles; a 4-stage smem ring (48 KB per
// stage at N = 256) and 2 x N TMEM columns let tile i's epilogue run under
// tile i+1's MMAs.  Reference: training.py:370-427.
#include "common.cuh"
#include "tc.cuh"

namespace dgnn {
using namespace tc;

namespace wsk {
constexpr int BM = 128;
constexpr int KC = 16;
constexpr int A_TILE = BM * 64;
constexpr int MAX_STAGES = 4;
// Bottleneck probe (scripts/ws_probe.cu builds with -DDGNN_WS_PROBE=mask):
// 1 skip MMAs, 2 zero-fill activations (no HBM reads), 4 skip weight copies,
// 8 epilogue without cell math / stores, 16 without stores, 32 without cell
// math.  Always 0 in the library.
#ifndef DGNN_WS_PROBE
#define DGNN_WS_PROBE 0
#endif
constexpr int PROBE = DGNN_WS_PROBE;
}  // namespace wsk

// Warp roles: NP producer warps, one MMA warp, NE epilogue warps (a multiple
// of 4 so every TMEM lane quarter has an owner).
template <int NP, int NE, int ST = 4, int EXTRA = 0>
struct WsRoles {
    static constexpr int NPROD = NP;
    static constexpr int MMA_WARP = NP;
    static constexpr int NEPI = NE;
    static constexpr int STAGES = ST;                    // A/B smem ring depth
    static constexpr int EXTRA_WARP = NP + 1 + NE;       // first warp after the epilogue
    static constexpr int THREADS = 32 * (NP + 1 + NE + EXTRA);
    static constexpr int NPT = 32 * NP;   // producer threads
};
// forward: heavy cell epilogue -- 16 epilogue warps (each a quarter of the
// units of its TMEM lane quarter) at hidden 32; at hidden 64, 8 (half the
// units each): 17 warps leave more registers per thread, 5-6% faster at
// configs[1] than 16 (scripts/fwd_roles.sh: 458 vs 481 us at kx 128)
#ifndef DGNN_FWD_NPROD
#define DGNN_FWD_NPROD 8
#endif
#ifndef DGNN_FWD_NEPI64
#define DGNN_FWD_NEPI64 8
#endif
#ifndef DGNN_FWD_NEPI32
#define DGNN_FWD_NEPI32 16
#endif
#ifndef DGNN_FWD_ST64
#define DGNN_FWD_ST64 3
#endif
#ifndef DGNN_FWD_RAW64
#define DGNN_FWD_RAW64 6
#endif
template <int HP>
using FwdRoles = WsRoles<DGNN_FWD_NPROD, (HP >= 64 ? DGNN_FWD_NEPI64 : (HP >= 32 ? DGNN_FWD_NEPI32 : 8)), (HP >= 64 ? DGNN_FWD_ST64 : 4)>;
// forward activation landing ring (fp32 chunks, cp.async), decoupled from
// the operand stages so loads run RAW_RING - 1 chunks ahead (6 at hidden 64:
// the operand stages are 48 KB and the c_prev tile takes 32 KB)
template <int HP>
constexpr int raw_ring() { return HP >= 64 ? DGNN_FWD_RAW64 : 8; }
// backward: 8 dz-producer warps fed from shared memory by one loader warp
// (the extra warp), 3-stage A/B ring to leave room for the raw input ring
#ifndef DGNN_BWD_NPROD
#define DGNN_BWD_NPROD 8
#endif
using BwdRoles = WsRoles<DGNN_BWD_NPROD, 4, 3, 1>;

__host__ __device__ constexpr int ws_tmem_cols(int n2) {
    return n2 <= 32 ? 32 : (n2 <= 64 ? 64 : (n2 <= 128 ? 128 : (n2 <= 256 ? 256 : 512)));
}

struct WsBars {
    uint64_t full_a[wsk::MAX_STAGES], full_b[wsk::MAX_STAGES], empty[wsk::MAX_STAGES], accfull[2], accempty[2];
    uint64_t raw_full[wsk::MAX_STAGES], raw_empty[wsk::MAX_STAGES];   // backward input ring
    uint64_t cp_full, cp_empty;                                         // forward c_prev tile
    uint32_t tmem;
};

// stage layout: [A hi | A lo | B hi+lo]
struct WsSmem {
    uint32_t base;   // smem address of stage 0 (1024-aligned)
    int stage;       // stage bytes
    __device__ uint32_t a_hi(int s) const { return base + s * stage; }
    __device__ uint32_t a_lo(int s) const { return base + s * stage + wsk::A_TILE; }
    __device__ uint32_t b(int s) const { return base + s * stage + 2 * wsk::A_TILE; }
};

template <class R>
inline size_t ws_smem_bytes(int n) {
    return (size_t)R::STAGES * (2 * wsk::A_TILE + 2 * n * 64) + 1024 + sizeof(WsBars) + 64;
}

template <class R>
__device__ __forceinline__ WsBars* ws_setup(WsSmem& sm, int n) {
    extern __shared__ uint8_t ws_smem_raw[];
    const uint32_t raw = smem_u32(ws_smem_raw);
    const uint32_t pad = (1024 - (raw & 1023)) & 1023;
    sm.base = raw + pad;
    sm.stage = 2 * wsk::A_TILE + 2 * n * 64;
    WsBars* bars = reinterpret_cast<WsBars*>(ws_smem_raw + pad + R::STAGES * sm.stage);
    const int warp = threadIdx.x >> 5;
    if (warp == R::MMA_WARP) tmem_alloc(&bars->tmem, ws_tmem_cols(2 * n));
    if (threadIdx.x == 0) {
        for (int s = 0; s < R::STAGES; ++s) {
            mbar_init(&bars->full_a[s], R::NPROD);
            mbar_init(&bars->full_b[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->accfull[a], 1);
            mbar_init(&bars->accempty[a], R::NEPI);
        }
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();
    return bars;
}

template <class R>
__device__ __forceinline__ void ws_teardown(WsBars* bars, int n) {
    fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == R::MMA_WARP) tmem_dealloc(bars->tmem, ws_tmem_cols(2 * n));
}

// MMA issuer: for every tile of this CTA, all K chunks into accumulator a.
template <class R>
__device__ __forceinline__ void ws_mma_loop(const WsSmem& sm, WsBars* bars, int n, int ntiles, int nch) {
    uint32_t gc = 0, it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const uint32_t a = it & 1, u = it >> 1;
        if (u >= 1) mbar_wait(&bars->accempty[a], (u - 1) & 1);
        fence_after();
        const uint32_t d = bars->tmem + a * n;
        for (int ch = 0; ch < nch; ++ch, ++gc) {
            const int s = gc % R::STAGES;
            const uint32_t j = gc / R::STAGES;
            mbar_wait(&bars->full_a[s], j & 1);
            mbar_wait(&bars->full_b[s], j & 1);
            fence_after();
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const uint64_t ahi = sdesc(sm.a_hi(s) + 32 * kk, 512, kSW64);
                const uint64_t alo = sdesc(sm.a_lo(s) + 32 * kk, 512, kSW64);
                for (int n0 = 0; n0 < n; n0 += 256) {
                    const int nn = n - n0 < 256 ? n - n0 : 256;
                    const uint32_t idesc = idesc_tf32(wsk::BM, nn);
                    const uint64_t bhi = sdesc(sm.b(s) + n0 * 64 + 32 * kk, 512, kSW64);
                    const uint64_t blo = sdesc(sm.b(s) + n * 64 + n0 * 64 + 32 * kk, 512, kSW64);
                    if (wsk::PROBE & 1) continue;
                    mma_tf32(d + n0, ahi, bhi, idesc, (ch == 0 && kk == 0) ? 0u : 1u);
                    mma_tf32(d + n0, ahi, blo, idesc, 1u);
                    mma_tf32(d + n0, alo, bhi, idesc, 1u);
                }
            }
            commit(&bars->empty[s]);
        }
        commit(&bars->accfull[a]);
    }
}

// Producer side of one chunk: wait for the stage, launch the weight copy,
// store the activation split.  `vals[i]` holds the 4 fp32 of item
// ptid + NPT i (row item / 4, column group item % 4).
template <class R, int ITEMS>
__device__ __forceinline__ void ws_produce(const WsSmem& sm, WsBars* bars, uint32_t gc, const float* img, int ch,
                                           uint32_t b_bytes, const float4 (&vals)[ITEMS]) {
    const int ptid = threadIdx.x;   // producers are threads 0 .. NPT-1
    const int s = gc % R::STAGES;
    const uint32_t j = gc / R::STAGES;
    if (j >= 1) mbar_wait(&bars->empty[s], (j - 1) & 1);
    if (ptid == 0) {
        mbar_arrive_expect_tx(&bars->full_b[s], b_bytes);
        bulk_g2s(sm.b(s), reinterpret_cast<const char*>(img) + (size_t)ch * b_bytes, b_bytes, &bars->full_b[s]);
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int idx = ptid + R::NPT * i;
        const int r = idx >> 2, q = idx & 3;
        float4 hi, lo;
        split4(vals[i], hi, lo);
        sts128(sm.a_hi(s) + sw64(r, q), hi);
        sts128(sm.a_lo(s) + sw64(r, q), lo);
    }
    fence_async_smem();
    __syncwarp();
    if ((ptid & 31) == 0) mbar_arrive(&bars->full_a[s]);
}

// ---------------------------------------------------------------------------
// forward

template <int HP>
__global__ void __launch_bounds__(FwdRoles<HP>::THREADS, 1) lstm_fwd_ws_kernel(
    int64_t rows, int kx, const float* __restrict__ x, int64_t ldx, const float* __restrict__ hprev,
    const float* __restrict__ cprev, const float* __restrict__ img, const float* __restrict__ bias,
    float* __restrict__ hout, float* __restrict__ cout, float* __restrict__ gates) {
    constexpr int N = 4 * HP;
    using R = FwdRoles<HP>;
    constexpr int ITEMS = wsk::BM * 4 / R::NPT;   // 4
    WsSmem sm;
    WsBars* bars = ws_setup<R>(sm, N);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (int)cdiv(rows, wsk::BM);
    const int K = kx + HP;
    const int nch = (K + wsk::KC - 1) / wsk::KC;
    const uint32_t b_bytes = 2 * N * 64;
    const uint32_t cpbuf = sm.base + R::STAGES * sm.stage + 1024 + raw_ring<HP>() * wsk::A_TILE;
    if (threadIdx.x == 0) {
        mbar_init(&bars->cp_full, 1);
        mbar_init(&bars->cp_empty, R::NEPI);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp < R::NPROD) {
        // Activations land (cp.async, fp32, SW64) in a raw ring RAW_RING
        // chunks deep, decoupled from the (few, 48 KB) operand stages: the
        // loads run up to RAW_RING - 1 chunks (56 KB) ahead, which covers
        // HBM latency at the MMA pace; the split writes the hi / lo operand
        // tiles once the stage is free.  Each producer thread loads, splits
        // and reloads only its own items, so a raw slot needs no barrier.
        constexpr int RS = raw_ring<HP>();
        const int ptid = threadIdx.x;
        const int my_tiles = blockIdx.x < ntiles ? (int)cdiv(ntiles - blockIdx.x, gridDim.x) : 0;
        const uint32_t G = (uint32_t)my_tiles * nch;
        const uint32_t raw0 = sm.base + R::STAGES * sm.stage + 1024;
        auto issue = [&](uint32_t g) {
            const int tile = blockIdx.x + (int)(g / nch) * gridDim.x;
            const int ch = (int)(g % nch);
            const uint32_t slot = raw0 + (g % RS) * wsk::A_TILE;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int idx = ptid + R::NPT * i;
                const int r = idx >> 2, q = idx & 3;
                const int64_t gr = (int64_t)tile * wsk::BM + r;
                const int k = ch * wsk::KC + 4 * q;
                const bool ok = gr < rows && k < K && !(wsk::PROBE & 2);
                const float* src = !ok ? x : (k < kx ? x + gr * ldx + k : hprev + gr * HP + (k - kx));
                cp_async16(slot + sw64(r, q), src, ok ? 16u : 0u);
            }
        };
        for (uint32_t g = 0; g < (uint32_t)(RS - 1); ++g) {
            if (g < G) issue(g);
            cp_async_commit();
        }
        for (uint32_t g = 0; g < G; ++g) {
            const int s = g % R::STAGES;
            const uint32_t j = g / R::STAGES;
            if (j >= 1) mbar_wait(&bars->empty[s], (j - 1) & 1);
            if (ptid == 0) {
                if (wsk::PROBE & 4) {
                    mbar_arrive(&bars->full_b[s]);
                } else {
                    const int ch = (int)(g % nch);
                    mbar_arrive_expect_tx(&bars->full_b[s], b_bytes);
                    bulk_g2s(sm.b(s), reinterpret_cast<const char*>(img) + (size_t)ch * b_bytes, b_bytes,
                             &bars->full_b[s]);
                }
            }
            cp_async_wait<RS - 2>();
            const uint32_t slot = raw0 + (g % RS) * wsk::A_TILE;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int idx = ptid + R::NPT * i;
                const uint32_t off = sw64(idx >> 2, idx & 3);
                float4 hi, lo;
                split4(lds128(slot + off), hi, lo);
                sts128(sm.a_hi(s) + off, hi);
                sts128(sm.a_lo(s) + off, lo);
            }
            fence_async_smem();
            __syncwarp();
            if ((ptid & 31) == 0) mbar_arrive(&bars->full_a[s]);
            if (g + RS - 1 < G) issue(g + RS - 1);
            cp_async_commit();
        }
    } else if (warp == R::MMA_WARP) {
        if (lane == 0) {
            ws_mma_loop<R>(sm, bars, N, ntiles, nch);
        } else if (lane == 1) {
            // c_prev is tile-blocked: a tile's rows are one contiguous block.
            // Bulk-copy it into shared memory as soon as the epilogue has read
            // the previous one, so the tile's cell update never waits on HBM.
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
                if (it >= 1) mbar_wait(&bars->cp_empty, (it - 1) & 1);
                const int64_t t0 = (int64_t)tile * wsk::BM;
                const uint32_t bytes = (uint32_t)((rows - t0 < wsk::BM ? rows - t0 : wsk::BM) * HP * 4);
                mbar_arrive_expect_tx(&bars->cp_full, bytes);
                bulk_g2s(cpbuf, cprev + t0 * HP, bytes, &bars->cp_full);
            }
        }
        __syncwarp();
    } else {
        const int e = warp - R::MMA_WARP - 1;
        constexpr int UPW = HP / (R::NEPI / 4);   // units per epilogue warp
        const int q = warp & 3, part = e >> 2;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const uint32_t a = it & 1, u = it >> 1;
            const int64_t row = (int64_t)tile * wsk::BM + 32 * q + lane;
            const int64_t t0 = (int64_t)tile * wsk::BM;
            const bool valid = row < rows;
            float cp[UPW];
            mbar_wait(&bars->cp_full, it & 1);
#pragma unroll
            for (int i = 0; i < UPW / 4; ++i) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (valid) v = lds128(cpbuf + 4 * (uint32_t)(tb_off(row, part * UPW + 4 * i, HP, rows) - t0 * HP));
                cp[4 * i] = v.x;
                cp[4 * i + 1] = v.y;
                cp[4 * i + 2] = v.z;
                cp[4 * i + 3] = v.w;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->cp_empty);
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
                if (!valid || (wsk::PROBE & 8)) continue;
                float hv[8], cv[8], gi[8], gf[8], go[8], gg[8];
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    if (wsk::PROBE & 32) {   // probe: stores without the cell math
                        gi[jj] = z[0][jj]; gf[jj] = z[1][jj]; go[jj] = z[2][jj]; gg[jj] = z[3][jj];
                        cv[jj] = z[0][jj] + cp[8 * g8 + jj]; hv[jj] = z[1][jj];
                        continue;
                    }
                    gi[jj] = act_sigmoid(z[0][jj] + __ldg(bias + 0 * HP + u0 + jj));
                    gf[jj] = act_sigmoid(z[1][jj] + __ldg(bias + 1 * HP + u0 + jj));
                    go[jj] = act_sigmoid(z[2][jj] + __ldg(bias + 2 * HP + u0 + jj));
                    gg[jj] = act_tanh(z[3][jj] + __ldg(bias + 3 * HP + u0 + jj));
                    cv[jj] = gf[jj] * cp[8 * g8 + jj] + gi[jj] * gg[jj];
                    hv[jj] = go[jj] * act_tanh(cv[jj]);
                }
                if (wsk::PROBE & 16) {   // probe: cell math without the stores
                    float acc = 0.f;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) acc += hv[jj] + cv[jj] + gi[jj] + gf[jj] + go[jj] + gg[jj];
                    if (acc == 12345.f) hout[row] = acc;
                    continue;
                }
                float4* ho = reinterpret_cast<float4*>(hout + row * HP + u0);
                ho[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
                ho[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
                // c and the gate cache are tile-blocked: 512 B per warp store
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
            if (lane == 0) mbar_arrive(&bars->accempty[a]);
        }
    }
    ws_teardown<R>(bars, N);
}

// ---------------------------------------------------------------------------
// backward: producers compute dz (unit-major K chunk = 4 units x 4 gates)

template <int HP>
__global__ void __launch_bounds__(BwdRoles::THREADS, 1) lstm_bwd_ws_kernel(
    int64_t rows, int kx, int N, const float* __restrict__ dy, const float* __restrict__ dh_in,
    const float* __restrict__ dc_in, float* gates, const float* __restrict__ cprev, const float* __restrict__ cnew,
    const float* __restrict__ img, float* __restrict__ dx, int64_t lddx, float* __restrict__ dh_out,
    float* __restrict__ dc_out) {
    constexpr int NC = 4 * HP;
    using R = BwdRoles;
    constexpr int ITEMS = wsk::BM * 4 / R::NPT;   // (row, unit) items per producer thread
    WsSmem sm;
    WsBars* bars = ws_setup<R>(sm, N);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = (int)cdiv(rows, wsk::BM);
    const int nch = HP / 4;
    const uint32_t b_bytes = 2 * N * 64;

    // raw input ring: per chunk (tile, 4 units) the 7 tile-blocked arrays
    // (gates i/f/o/g, c_prev, c_new, dc_in: one contiguous tr x 16 B block
    // each, bulk-copied) and the row-major dh_in / dy pieces (cp.async)
    constexpr int RAWF = wsk::BM * 4 * 9;              // floats per slot
    const int RSLOTS = N > 192 ? 3 : 4;                 // what fits next to the A/B ring
    constexpr int O_CP = 4 * 512, O_CN = 5 * 512, O_DC = 6 * 512, O_DH = 7 * 512, O_DY = 8 * 512;
    const uint32_t raw0 = sm.base + R::STAGES * sm.stage + 1024 + R::NEPI * 4096;
    const float* rawf = reinterpret_cast<const float*>(
        reinterpret_cast<const uint8_t*>(bars) + (raw0 - smem_u32(bars)));
    const int my_tiles = blockIdx.x < ntiles ? (int)cdiv(ntiles - blockIdx.x, gridDim.x) : 0;
    const uint32_t G = (uint32_t)my_tiles * nch;
    if (threadIdx.x == 0) {
        for (int i = 0; i < RSLOTS; ++i) {
            mbar_init(&bars->raw_full[i], 33);             // 32 cp.async lanes + the expect_tx arrival
            mbar_init(&bars->raw_empty[i], R::NPROD);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == R::EXTRA_WARP) {
        // loader: stays up to RSLOTS chunks ahead of the dz producers
        for (uint32_t g = 0; g < G; ++g) {
            const int tile = blockIdx.x + (int)(g / nch) * gridDim.x, ch = (int)(g % nch);
            const int slot = g % RSLOTS;
            const uint32_t j = g / RSLOTS;
            if (j >= 1) mbar_wait_sleep(&bars->raw_empty[slot], (j - 1) & 1);
            const uint32_t rb = raw0 + slot * RAWF * 4;
            const int64_t t0 = (int64_t)tile * wsk::BM;
            const int tr = (int)min((int64_t)wsk::BM, rows - t0);
            const uint32_t blk = (uint32_t)tr * 16;
            if (lane == 0) {
                mbar_arrive_expect_tx(&bars->raw_full[slot], 7 * blk);
#pragma unroll
                for (int gg = 0; gg < 4; ++gg)
                    bulk_g2s(rb + gg * 2048, gates + tb_off(t0, gg * HP + 4 * ch, NC, rows), blk, &bars->raw_full[slot]);
                bulk_g2s(rb + O_CP * 4, cprev + tb_off(t0, 4 * ch, HP, rows), blk, &bars->raw_full[slot]);
                bulk_g2s(rb + O_CN * 4, cnew + tb_off(t0, 4 * ch, HP, rows), blk, &bars->raw_full[slot]);
                bulk_g2s(rb + O_DC * 4, dc_in + tb_off(t0, 4 * ch, HP, rows), blk, &bars->raw_full[slot]);
            }
#pragma unroll
            for (int r = lane; r < wsk::BM; r += 32) {
                const int64_t row = t0 + r;
                const bool ok = r < tr;
                cp_async16(rb + (O_DH + 4 * r) * 4, ok ? dh_in + row * HP + 4 * ch : dh_in, ok ? 16u : 0u);
                cp_async16(rb + (O_DY + 4 * r) * 4, (ok && dy) ? dy + row * HP + 4 * ch : dh_in, (ok && dy) ? 16u : 0u);
            }
            cp_async_mbar_arrive(&bars->raw_full[slot]);
        }
        cp_async_wait<0>();
    } else if (warp < R::NPROD) {
        const int ptid = threadIdx.x;
        for (uint32_t g = 0; g < G; ++g) {
            const int tile = blockIdx.x + (int)(g / nch) * gridDim.x, ch = (int)(g % nch);
            const int slot = g % RSLOTS;
            mbar_wait(&bars->raw_full[slot], (g / RSLOTS) & 1);
            const float* rw = rawf + slot * RAWF;
            float4 vals[ITEMS];
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const int idx = ptid + R::NPT * i;   // = 4 r + uu: the slot's [r][uu] order
                const int64_t row = (int64_t)tile * wsk::BM + (idx >> 2);
                const int u = 4 * ch + (idx & 3);
                float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                if (row < rows) {
                    const float gi = rw[idx], gf = rw[512 + idx], go = rw[1024 + idx], gg = rw[1536 + idx];
                    const float cpv = rw[O_CP + idx], cn = rw[O_CN + idx], dcv = rw[O_DC + idx];
                    const float dhv = rw[O_DY + idx] + rw[O_DH + idx];
                    const float tcn = act_tanh(cn);
                    const float d_o = dhv * tcn;
                    const float dc = dhv * go * (1.f - tcn * tcn) + dcv;
                    const float df = dc * cpv, di = dc * gg, dg = dc * gi;
                    dc_out[tb_off(row, u, HP, rows)] = dc * gf;
                    z = make_float4(di * gi * (1.f - gi), df * gf * (1.f - gf), d_o * go * (1.f - go), dg * (1.f - gg * gg));
                    // dz replaces the gate cache
                    gates[tb_off(row, u, NC, rows)] = z.x;
                    gates[tb_off(row, HP + u, NC, rows)] = z.y;
                    gates[tb_off(row, 2 * HP + u, NC, rows)] = z.z;
                    gates[tb_off(row, 3 * HP + u, NC, rows)] = z.w;
                }
                vals[i] = z;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->raw_empty[slot]);
            ws_produce<R, ITEMS>(sm, bars, g, img, ch, b_bytes, vals);
        }
    } else if (warp == R::MMA_WARP) {
        if (lane == 0) ws_mma_loop<R>(sm, bars, N, ntiles, nch);
        __syncwarp();
    } else {
        // One warp per TMEM lane quarter.  [dx | dh] rows go out through a
        // per-warp shared-memory transpose, 32 columns at a time: each warp
        // store then covers 4 rows x 128 contiguous bytes instead of 32 rows
        // x 16 B.
        static_assert(R::NEPI == 4, "one epilogue warp per lane quarter");
        const int e = warp - R::MMA_WARP - 1;
        const int q = warp & 3;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const uint32_t ebuf = sm.base + R::STAGES * sm.stage + 1024 + e * 4096;
        const int K = kx + HP;
        uint32_t it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const uint32_t a = it & 1, u = it >> 1;
            mbar_wait(&bars->accfull[a], u & 1);
            fence_after();
            const uint32_t tq = bars->tmem + lane_off + a * N;
            for (int c0 = 0; c0 < N; c0 += 32) {
                float v[4][8];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (c0 + 8 * j < N) tmem_ld8(tq + c0 + 8 * j, v[j]);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        sts128(ebuf + lane * 128 + ((((2 * j + h) ^ (lane & 7))) << 4),
                               make_float4(v[j][4 * h], v[j][4 * h + 1], v[j][4 * h + 2], v[j][4 * h + 3]));
                __syncwarp();
#pragma unroll
                for (int r0 = 0; r0 < 32; r0 += 4) {
                    const int r = r0 + (lane >> 3), ch = lane & 7;
                    const float4 val = lds128(ebuf + r * 128 + ((ch ^ (r & 7)) << 4));
                    const int64_t row = (int64_t)tile * wsk::BM + 32 * q + r;
                    const int c = c0 + 4 * ch;
                    if (row < rows) {
                        if (c < kx) *reinterpret_cast<float4*>(dx + row * lddx + c) = val;
                        else if (c < K) *reinterpret_cast<float4*>(dh_out + row * HP + (c - kx)) = val;
                    }
                }
                __syncwarp();
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->accempty[a]);
        }
    }
    ws_teardown<R>(bars, N);
}

template <int HP>
int lstm_fwd_ws_t(int64_t rows, int kx, const float* x, int64_t ldx, const float* hp_, const float* cp,
                  const float* img, const float* b, float* h, float* c, float* gates, cudaStream_t st) {
    constexpr int N = 4 * HP;
    auto k = lstm_fwd_ws_kernel<HP>;
    const size_t smem = ws_smem_bytes<FwdRoles<HP>>(N) + 1024 + (size_t)raw_ring<HP>() * wsk::A_TILE +
                        (size_t)wsk::BM * HP * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int ntiles = (int)cdiv(rows, wsk::BM);
    const int grid = ntiles < persistent_ctas() ? ntiles : persistent_ctas();
    note_launch();
    k<<<grid, FwdRoles<HP>::THREADS, smem, st>>>(rows, kx, x, ldx, hp_, cp, img, b, h, c, gates);
    return launch_status("lstm_forward_step_ws");
}

template <int HP>
int lstm_bwd_ws_t(int64_t rows, int kx, const float* dy, const float* dh_in, const float* dc_in, float* gates,
                  const float* cp, const float* cn, const float* img, float* dx, int64_t lddx, float* dh_out,
                  float* dc_out, cudaStream_t st) {
    const int N = (kx + HP + 15) / 16 * 16;
    if (N > 256) {
        set_error("lstm_backward_step: kx + hp = %d exceeds 256", kx + HP);
        return DGNN_EUNSUPPORTED;
    }
    auto k = lstm_bwd_ws_kernel<HP>;
    // + epilogue transpose buffers + the raw input ring (18 KB slots)
    const size_t smem = ws_smem_bytes<BwdRoles>(N) + 1024 + BwdRoles::NEPI * 4096 +
                        (size_t)(N > 192 ? 3 : 4) * wsk::BM * 4 * 9 * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int ntiles = (int)cdiv(rows, wsk::BM);
    const int grid = ntiles < persistent_ctas() ? ntiles : persistent_ctas();
    note_launch();
    k<<<grid, BwdRoles::THREADS, smem, st>>>(rows, kx, N, dy, dh_in, dc_in, gates, cp, cn, img, dx, lddx, dh_out,
                                         dc_out);
    return launch_status("lstm_backward_step_ws");
}

}  // namespace dgnn

using namespace dgnn;

extern "C" {

int dgnn_lstm_forward_step_ws(int64_t rows, int32_t kx, int32_t hp, const float* x, int64_t ldx,
                              const float* h_prev, const float* c_prev, const float* wimg, const float* bias,
                              float* h_out, float* c_out, float* gates, void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && kx % 4 == 0 && ldx % 4 == 0, "lstm_forward_step_ws: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 16: return lstm_fwd_ws_t<16>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
        case 32: return lstm_fwd_ws_t<32>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
        case 64: return lstm_fwd_ws_t<64>(rows, kx, x, ldx, h_prev, c_prev, wimg, bias, h_out, c_out, gates, st);
    }
    set_error("lstm_forward_step_ws: unsupported hp %d (use dgnn_lstm_forward_step_tc)", hp);
    return DGNN_EUNSUPPORTED;
}

int dgnn_lstm_backward_step_ws(int64_t rows, int32_t kx, int32_t hp, const float* dy, const float* dh_in,
                               const float* dc_in, float* gates, const float* c_prev, const float* c_new,
                               const float* wimg, float* dx, int64_t lddx, float* dh_out, float* dc_out,
                               void* stream) {
    DGNN_CHECK_ARG(rows >= 0 && kx % 4 == 0 && lddx % 4 == 0, "lstm_backward_step_ws: bad sizes");
    if (rows == 0) return DGNN_OK;
    cudaStream_t st = as_stream(stream);
    switch (hp) {
        case 16: return lstm_bwd_ws_t<16>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wimg, dx, lddx, dh_out, dc_out, st);
        case 32: return lstm_bwd_ws_t<32>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wimg, dx, lddx, dh_out, dc_out, st);
        case 64: return lstm_bwd_ws_t<64>(rows, kx, dy, dh_in, dc_in, gates, c_prev, c_new, wimg, dx, lddx, dh_out, dc_out, st);
    }
    set_error("lstm_backward_step_ws: unsupported hp %d (use dgnn_lstm_backward_step_tc)", hp);
    return DGNN_EUNSUPPORTED;
}

}  // extern "C"
