// tile_pattern_bw.cu -- HBM bandwidth of an in-place read+write sweep over
// 2^n complex128 amplitudes as a function of the tile's bit set (the access
// pattern of a tile pass without its arithmetic): a tile = the 2^K
// amplitudes whose bits outside T are fixed; T = the low C bits (128-byte
// runs for C = 3) + K - C contiguous bits starting at `hi`.  Each CTA owns
// whole tiles (persistent grid), each thread moves U amplitudes of a tile
// (loads first, then stores).  Prints GB/s (read + write bytes) per pattern.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tpbw tools/tile_pattern_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int U = 16;

__device__ __forceinline__ uint64_t tile_addr(uint64_t tile, uint32_t l, int C, int hi, int K) {
    // l: K-bit in-tile index (low C bits, then K - C bits placed at hi);
    // tile: the free bits in order (bits [C, hi) then [hi + K - C, n))
    const uint64_t lo = l & ((1u << C) - 1), mid = l >> C;
    const int gap = hi - C;
    const uint64_t t_lo = tile & ((1ull << gap) - 1), t_hi = tile >> gap;
    return lo | (t_lo << C) | (mid << hi) | (t_hi << (hi + K - C));
}

__global__ void __launch_bounds__(128) sweep(double2 *__restrict__ s, uint64_t n_tiles, int K, int C, int hi) {
    const uint32_t T = 1u << K, per = T / U;   // threads per tile
    const uint32_t lane = threadIdx.x % per, slot = threadIdx.x / per, tiles_per_cta = blockDim.x / per;
    for (uint64_t t = (uint64_t)blockIdx.x * tiles_per_cta + slot; t < n_tiles; t += (uint64_t)gridDim.x * tiles_per_cta) {
        double2 a[U];
        uint64_t ad[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            ad[u] = tile_addr(t, lane + u * per, C, hi, K);
            a[u] = s[ad[u]];
        }
#pragma unroll
        for (int u = 0; u < U; u++) s[ad[u]] = make_double2(a[u].y, a[u].x);
    }
}

int main() {
    const int n = 28;
    const uint64_t N = 1ull << n;
    double2 *s;
    if (cudaMalloc(&s, N * sizeof(double2)) != cudaSuccess) return 1;
    cudaMemset(s, 0, N * sizeof(double2));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int K = 11;
    int cs[] = {3, 3, 3, 3, 3, 4, 5, 11};
    int his[] = {3, 8, 12, 17, 20, 20, 20, 11};
    for (int i = 0; i < 8; i++) {
        const int C = cs[i], hi = his[i] < C ? C : his[i];
        const uint64_t n_tiles = N >> K;
        for (int occ : {4, 8, 16}) {
            const int grid = sms * occ;
            sweep<<<grid, 128>>>(s, n_tiles, K, C, hi);
            cudaEventRecord(a);
            const int R = 5;
            for (int r = 0; r < R; r++) sweep<<<grid, 128>>>(s, n_tiles, K, C, hi);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double gbs = 32.0 * N * R / (ms * 1e-3) / 1e9;
            printf("{\"K\": %d, \"C\": %d, \"hi\": %d, \"ctas_per_sm\": %d, \"GBps\": %.1f, \"ms\": %.3f}\n", K, C, hi,
                   occ, gbs, ms / R);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
