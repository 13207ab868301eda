// tile_pattern_bw.cu -- HBM bandwidth of an in-place read+write sweep over
// complex128 amplitudes as a function of the tile's bit set: the access
// pattern of a tile pass without its arithmetic.  A tile = the 2^K
// amplitudes whose bits outside the tile set T are fixed; each CTA owns
// whole tiles (persistent grid, tiles in the order of their free bits, as
// the tile kernel), each thread moves U amplitudes of a tile (loads first,
// then stores).  Prints GB/s of read + write bytes.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tpbw tools/tile_pattern_bw.cu
//   /tmp/tpbw                      # built-in sweep: 128-B runs + 8 contiguous bits at increasing strides
//   /tmp/tpbw masks N MASK...      # N index bits (e.g. 26 = 4 circuits of 2^24), one hex tile mask per pass
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int U = 16;

struct Pattern {
    int K, nfree;
    uint8_t tpos[16];   // tile bit positions, ascending
    uint8_t fpos[48];   // free bit positions, ascending
};

__device__ __forceinline__ uint64_t deposit(uint64_t v, const uint8_t *pos, int cnt) {
    uint64_t a = 0;
    for (int i = 0; i < cnt; i++) a |= ((v >> i) & 1ull) << pos[i];
    return a;
}

// pf = 0: plain.  pf = B > 0: before loading a tile, the threads holding the
// first amplitude of each 128-byte run also ask L2 for the B-byte aligned
// block around it (cp.async.bulk.prefetch.L2) -- runs of the neighbouring
// tiles, which other CTAs load at about the same time.  pf = -B: the same
// for the NEXT tile this CTA will process.
template <int MAXT>
__global__ void __launch_bounds__(MAXT) sweep(double2 *__restrict__ s, uint64_t n_tiles, Pattern P, int pf) {
    const uint32_t T = 1u << P.K, per = T / U;   // threads per tile
    const uint32_t lane = threadIdx.x % per, slot = threadIdx.x / per, tiles_per_cta = blockDim.x / per;
    uint64_t off[U];
#pragma unroll
    for (int u = 0; u < U; u++) off[u] = deposit(lane + u * per, P.tpos, P.K);
    const uint64_t step = (uint64_t)gridDim.x * tiles_per_cta;
    const uint32_t pb = pf < 0 ? -pf : pf;
    for (uint64_t t = (uint64_t)blockIdx.x * tiles_per_cta + slot; t < n_tiles; t += step) {
        const uint64_t base = deposit(t, P.fpos, P.nfree);
        if (pf != 0) {
            const uint64_t tp = pf > 0 ? t : t + step;
            if (tp < n_tiles) {
                const uint64_t bp = pf > 0 ? base : deposit(tp, P.fpos, P.nfree);
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (((bp | off[u]) & 7) == 0) {
                        const uint64_t a = (uint64_t)(s + (bp | off[u])) & ~(uint64_t)(pb - 1);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(pb) : "memory");
                    }
            }
        }
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; u++) a[u] = s[base | off[u]];
#pragma unroll
        for (int u = 0; u < U; u++) s[base | off[u]] = make_double2(a[u].y, a[u].x);
    }
}

// TPBW_PAIR = 1 / 2: clusters of two CTAs sweep adjacent tiles (t, t + 1: the
// 128-byte runs of one are the neighbours of the other's) in lockstep -- a
// cluster barrier before each tile's loads (1) and also before its stores
// (2) -- to see whether HBM serves two 128-byte halves of a 256-byte segment
// that arrive from two SMs at about the same time like one 256-byte run.
template <int MAXT>
__global__ void __launch_bounds__(MAXT) sweep_pair(double2 *__restrict__ s, uint64_t n_tiles, Pattern P, int mode) {
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t T = 1u << P.K, per = T / U;
    const uint32_t lane = threadIdx.x % per, slot = threadIdx.x / per, tiles_per_cta = blockDim.x / per;
    uint64_t off[U];
#pragma unroll
    for (int u = 0; u < U; u++) off[u] = deposit(lane + u * per, P.tpos, P.K);
    const uint64_t step = (uint64_t)gridDim.x * tiles_per_cta;
    // (trip counts agree inside a cluster: n_tiles and the grid are even)
    for (uint64_t t = (uint64_t)blockIdx.x * tiles_per_cta + slot; t < n_tiles; t += step) {
        const uint64_t base = deposit(t, P.fpos, P.nfree);
        cl.sync();
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; u++) a[u] = s[base | off[u]];
        if (mode >= 2) cl.sync();
#pragma unroll
        for (int u = 0; u < U; u++) s[base | off[u]] = make_double2(a[u].y, a[u].x);
    }
}

static Pattern make(int n, uint64_t mask) {
    Pattern P{};
    for (int b = 0; b < n; b++) {
        if (mask >> b & 1) P.tpos[P.K++] = (uint8_t)b;
        else P.fpos[P.nfree++] = (uint8_t)b;
    }
    return P;
}

static double run(double2 *s, int n, uint64_t mask, int occ, int sms, float *ms_out, int pf = 0) {
    Pattern P = make(n, mask);
    const uint64_t n_tiles = 1ull << P.nfree;
    const int threads = (1 << P.K) / U > 128 ? (1 << P.K) / U : 128;
    const int grid = sms * occ * 128 / threads;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // 13-bit tiles (512 threads) get their own instantiation, so the 256-thread
    // code the earlier measurements used is unchanged
    const int pair = getenv("TPBW_PAIR") ? atoi(getenv("TPBW_PAIR")) : 0;
    auto launch = [&]() {
        if (pair && threads <= 256 && threads == (1 << P.K) / U) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid & ~1);
            cfg.blockDim = dim3(threads);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, sweep_pair<256>, s, n_tiles, P, pair);
        } else if (threads <= 256) sweep<256><<<grid, threads>>>(s, n_tiles, P, pf);
        else sweep<512><<<grid, threads>>>(s, n_tiles, P, pf);
    };
    launch();
    cudaEventRecord(a);
    const int R = 5;
    for (int r = 0; r < R; r++) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_out = ms / R;
    return 32.0 * (double)(1ull << n) * R / (ms * 1e-3) / 1e9;
}

int main(int argc, char **argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 2 && std::string(argv[1]) == "masks") {
        const int n = atoi(argv[2]);
        double2 *s;
        if (cudaMalloc(&s, (16ull << n)) != cudaSuccess) return 1;
        cudaMemset(s, 0, 16ull << n);
        const int pf = getenv("TPBW_PF") ? atoi(getenv("TPBW_PF")) : 0;
        for (int i = 3; i < argc; i++) {
            const uint64_t mask = strtoull(argv[i], nullptr, 16);
            float ms = 0;
            const double g = run(s, n, mask, 16, sms, &ms, pf);
            printf("{\"n\": %d, \"mask\": \"0x%llx\", \"ctas_per_sm\": 16, \"l2_prefetch\": %d, \"GBps\": %.1f, \"ms\": %.4f}\n", n,
                   (unsigned long long)mask, pf, g, ms);
        }
        return 0;
    }
    const int n = 28;
    double2 *s;
    if (cudaMalloc(&s, 16ull << n) != cudaSuccess) return 1;
    cudaMemset(s, 0, 16ull << n);
    const int K = 11;
    int cs[] = {3, 3, 3, 3, 3, 4, 5, 11};
    int his[] = {3, 8, 12, 17, 20, 20, 20, 11};
    for (int i = 0; i < 8; i++) {
        const int C = cs[i], hi = his[i] < C ? C : his[i];
        uint64_t mask = (1ull << C) - 1;
        for (int b = 0; b < K - C; b++) mask |= 1ull << (hi + b);
        for (int occ : {4, 8, 16}) {
            float ms = 0;
            const double g = run(s, n, mask, occ, sms, &ms);
            printf("{\"K\": %d, \"C\": %d, \"hi\": %d, \"ctas_per_sm\": %d, \"GBps\": %.1f, \"ms\": %.3f}\n", K, C, hi,
                   occ, g, ms);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
