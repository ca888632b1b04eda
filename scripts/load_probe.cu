// Per-SM streaming-load probe: one persistent CTA per SM streams a large
// buffer from HBM into a shared-memory ring of `stages` x `stage_kb` KB,
// with (a) cp.async 16 B per thread (LDGSTS, mbarrier completion) or
// (b) cp.async.bulk (one elected thread, complete_tx), and a consumer warp
// group that only acknowledges each stage.  Reports GB/s against bytes in
// flight per SM, to tell whether thread-issued loads or the bulk-copy
// engine reach HBM rate at the ring depths the kernels here can afford.
// Build/run: scripts/load_probe.sh
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2109_07893_b200/csrc/tc.cuh"

using namespace dgnn::tc;

template <int MODE>   // 0 = LDGSTS, 1 = bulk
__global__ void __launch_bounds__(384, 1) stream_kernel(const uint8_t* __restrict__ src, int64_t bytes_per_cta,
                                                        int stages, int stage_bytes, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NLOAD = 8;   // loader warps (LDGSTS mode); warp 0 alone in bulk mode
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) {
            mbar_init(&full[i], MODE == 0 ? 32 * NLOAD : 1);
            mbar_init(&empty[i], 4);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const uint8_t* base = src + (int64_t)blockIdx.x * bytes_per_cta;
    const int nst = (int)(bytes_per_cta / stage_bytes);
    const uint32_t s0 = smem_u32(smem);
    if (warp < NLOAD) {
        if (MODE == 1 && warp > 0) return;
        for (int g = 0; g < nst; ++g) {
            const int s = g % stages, u = g / stages;
            if (u >= 1) mbar_wait(&empty[s], (u - 1) & 1);
            const uint8_t* p = base + (int64_t)g * stage_bytes;
            if (MODE == 0) {
                for (int o = threadIdx.x * 16; o < stage_bytes; o += 32 * NLOAD * 16)
                    cp_async16(s0 + s * stage_bytes + o, p + o, 16u);
                cp_async_mbar_arrive(&full[s]);
            } else if (lane == 0) {
                mbar_arrive_expect_tx(&full[s], stage_bytes);
                for (int o = 0; o < stage_bytes; o += 4096)
                    bulk_g2s(s0 + s * stage_bytes + o, p + o, min(4096, stage_bytes - o), &full[s]);
            }
        }
        if (MODE == 0) cp_async_wait<0>();
    } else if (warp < NLOAD + 4) {
        unsigned long long acc = 0;
        for (int g = 0; g < nst; ++g) {
            const int s = g % stages;
            mbar_wait(&full[s], (g / stages) & 1);
            acc += *reinterpret_cast<const uint32_t*>(smem + s * stage_bytes + 4 * lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 0x1234567) sink[0] = acc;
    }
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int64_t per = 64ll << 20;   // 64 MB per CTA, 9.5 GB total
    uint8_t* buf;
    if (cudaMalloc(&buf, per * nsm) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(buf, 1, per * nsm);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int kbs[] = {8, 16, 32};
    const int depths[] = {2, 3, 4, 6, 8, 12};
    for (int mode = 0; mode < 2; ++mode)
        for (int kb : kbs)
            for (int st : depths) {
                const int sb = kb * 1024;
                const size_t smem = (size_t)st * sb + 512;
                if (smem > 227 * 1024) continue;
                auto k = mode == 0 ? stream_kernel<0> : stream_kernel<1>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                const int64_t bytes = (per / sb) * sb;
                k<<<nsm, 384, smem>>>(buf, bytes, st, sb, sink);
                cudaEventRecord(e0);
                k<<<nsm, 384, smem>>>(buf, bytes, st, sb, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("%s stage %2d KB x %2d = %3d KB in flight/SM: %7.0f GB/s  %s\n", mode ? "bulk  " : "LDGSTS", kb,
                       st, kb * st, (double)bytes * nsm / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
