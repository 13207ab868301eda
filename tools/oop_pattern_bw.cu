// oop_pattern_bw.cu -- HBM bandwidth of an OUT-OF-PLACE tile sweep that reads
// each tile as 2^K contiguous amplitudes (bits 0..K-1) and writes it under a
// bit permutation: the tile's local bits 0..C-1 stay at 0..C-1 (runs of 2^C
// amplitudes), its local bits C..K-1 go to K-C positions starting at bit
// `hi`, and the free bits fill the remaining positions in order.  This is the
// access pattern of a pass that fuses the relabelling of the next pass's
// qubits into its store; compared with the in-place strided sweep of
// tile_pattern_bw.cu (same tile set on both sides).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/oopbw tools/oop_pattern_bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int U = 16;

struct Map {
    int n;
    uint8_t pos[48];   // new position of old bit b
};

__device__ __forceinline__ uint64_t permute(uint64_t v, const Map &M) {
    uint64_t a = 0;
    for (int i = 0; i < M.n; i++) a |= ((v >> i) & 1ull) << M.pos[i];
    return a;
}

// mode 0: out of place, read contiguous, write permuted
// mode 1: out of place, read permuted, write contiguous
// mode 2: in place, read + write permuted (the current tile pass)
__global__ void __launch_bounds__(256) sweep(const double2 *__restrict__ src, double2 *__restrict__ dst, uint64_t n_tiles,
                                             int K, Map M, int mode) {
    const uint32_t T = 1u << K, per = T / U;
    const uint32_t lane = threadIdx.x % per, slot = threadIdx.x / per, tiles_per_cta = blockDim.x / per;
    const uint64_t step = (uint64_t)gridDim.x * tiles_per_cta;
    uint64_t lp[U];
#pragma unroll
    for (int u = 0; u < U; u++) lp[u] = permute(lane + u * per, M);
    for (uint64_t t = (uint64_t)blockIdx.x * tiles_per_cta + slot; t < n_tiles; t += step) {
        double2 a[U];
        uint64_t c[U], p[U];
        const uint64_t bp = permute(t << K, M);
#pragma unroll
        for (int u = 0; u < U; u++) {
            c[u] = (t << K) | (lane + u * per);
            p[u] = bp | lp[u];
        }
        if (mode == 0) {
#pragma unroll
            for (int u = 0; u < U; u++) a[u] = src[c[u]];
#pragma unroll
            for (int u = 0; u < U; u++) dst[p[u]] = make_double2(a[u].y, a[u].x);
        } else if (mode == 1) {
#pragma unroll
            for (int u = 0; u < U; u++) a[u] = src[p[u]];
#pragma unroll
            for (int u = 0; u < U; u++) dst[c[u]] = make_double2(a[u].y, a[u].x);
        } else {
            double2 *s = dst;
#pragma unroll
            for (int u = 0; u < U; u++) a[u] = s[p[u]];
#pragma unroll
            for (int u = 0; u < U; u++) s[p[u]] = make_double2(a[u].y, a[u].x);
        }
    }
}

int main(int argc, char **argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = argc > 1 ? atoi(argv[1]) : 28;
    const int K = 11;
    double2 *a, *bb;
    if (cudaMalloc(&a, 16ull << n) != cudaSuccess || cudaMalloc(&bb, 16ull << n) != cudaSuccess) return 1;
    cudaMemset(a, 0, 16ull << n);
    cudaMemset(bb, 0, 16ull << n);
    int cs[] = {3, 3, 3, 3, 4, 5, 3, 4};
    int his[] = {8, 12, 17, 20, 20, 20, 14, 14};
    for (int i = 0; i < 8; i++) {
        const int C = cs[i], hi = his[i];
        Map M{};
        M.n = n;
        // new positions of the tile's local bits
        bool used[64] = {};
        if (hi + K - C > n) continue;
        for (int b = 0; b < C; b++) { M.pos[b] = b; used[b] = true; }
        for (int b = C; b < K; b++) { M.pos[b] = hi + (b - C); used[hi + (b - C)] = true; }
        int nxt = 0;
        for (int b = K; b < n; b++) {
            while (used[nxt]) nxt++;
            M.pos[b] = nxt;
            used[nxt] = true;
        }
        for (int mode = 0; mode < 3; mode++) {
            const int threads = 256, occ = 8;
            const int grid = sms * occ;
            const uint64_t n_tiles = 1ull << (n - K);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            sweep<<<grid, threads>>>(a, bb, n_tiles, K, M, mode);
            cudaEventRecord(e0);
            const int R = 6;
            for (int r = 0; r < R; r++) {
                if (r & 1) sweep<<<grid, threads>>>(bb, a, n_tiles, K, M, mode);
                else sweep<<<grid, threads>>>(a, bb, n_tiles, K, M, mode);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double g = 32.0 * (double)(1ull << n) * R / (ms * 1e-3) / 1e9;
            printf("{\"n\": %d, \"K\": %d, \"C\": %d, \"hi\": %d, \"mode\": \"%s\", \"GBps\": %.1f, \"ms\": %.4f}\n", n, K, C,
                   hi, mode == 0 ? "read_contig_write_perm" : mode == 1 ? "read_perm_write_contig" : "inplace_perm", g,
                   ms / R);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
