// tma_pattern_bw.cu -- does TMA move a strided tile faster than per-thread
// loads?  In-place read + write sweep of 2^n complex128 amplitudes, tile =
// the low C bits (one contiguous run of 2^C amplitudes) + K - C contiguous
// bits starting at `hi` (the tile shapes of tools/tile_pattern_bw.cu), one
// tile per CTA iteration over a persistent grid, staged through shared
// memory (double-buffered, 2^K amplitudes per buffer) like the tile kernel:
//   mode 0: per-thread cp.async (LDGSTS, 16 B) into smem, per-thread STG out
//   mode 1: one TMA 4-D tensor load (cp.async.bulk.tensor, mbarrier
//           completion) into smem, TMA tensor store out
// Prints GB/s of read + write bytes per (mode, pattern, CTAs per SM).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/tmabw tools/tma_pattern_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

constexpr int K = 11, T = 1 << K;   // amplitudes per tile (32 KiB)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Shape {
    int n, C, hi;
};

__device__ __forceinline__ uint64_t tile_base(uint64_t t, const Shape &s) {
    // free bits: [C, hi) then [hi + K - C, n)
    const int gap = s.hi - s.C;
    const uint64_t lo = t & ((1ull << gap) - 1), up = t >> gap;
    return (lo << s.C) | (up << (s.hi + K - s.C));
}
__device__ __forceinline__ uint64_t in_tile(uint32_t l, const Shape &s) {
    const uint64_t lo = l & ((1u << s.C) - 1), mid = l >> s.C;
    return lo | (mid << s.hi);
}

// mode 0: LDGSTS double buffer, STG stores (128 threads, 16 amplitudes each)
__global__ void __launch_bounds__(128) sweep_ldgsts(double2 *s, uint64_t n_tiles, Shape sh) {
    extern __shared__ double2 buf[];
    const uint32_t t = threadIdx.x;
    auto issue = [&](uint64_t g, double2 *b) {
        const uint64_t base = tile_base(g, sh);
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const uint32_t l = t + u * 128;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(b + l)), "l"(s + (base | in_tile(l, sh))));
        }
        asm volatile("cp.async.commit_group;");
    };
    uint64_t g = blockIdx.x;
    if (g >= n_tiles) return;
    issue(g, buf);
    for (int i = 0; g < n_tiles; i++, g += gridDim.x) {
        double2 *b = buf + (i & 1) * T;
        const uint64_t gn = g + gridDim.x;
        if (gn < n_tiles) issue(gn, buf + ((i + 1) & 1) * T);
        else asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 1;");
        __syncthreads();
        const uint64_t base = tile_base(g, sh);
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const uint32_t l = t + u * 128;
            const double2 v = b[l];
            s[base | in_tile(l, sh)] = make_double2(v.y, v.x);
        }
        __syncthreads();
    }
}

// mode 1: TMA tensor load / store, one elected thread, mbarrier per buffer
__global__ void __launch_bounds__(128) sweep_tma(const __grid_constant__ CUtensorMap tm, uint64_t n_tiles, Shape sh) {
    extern __shared__ __align__(1024) double2 buf[];
    __shared__ __align__(8) uint64_t bar[2];
    const uint32_t t = threadIdx.x;
    const int gap = sh.hi - sh.C;
    auto coords = [&](uint64_t g, int *c) {
        c[0] = 0;
        c[1] = (int)(g & ((1ull << gap) - 1));
        c[2] = 0;
        c[3] = (int)(g >> gap);
    };
    auto load = [&](uint64_t g, int slot) {
        int c[4];
        coords(g, c);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[slot])), "r"(T * 16));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                smem_u32(buf + slot * T)),
            "l"(&tm), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(smem_u32(&bar[slot]))
            : "memory");
    };
    uint64_t g = blockIdx.x;
    if (g >= n_tiles) return;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (t == 0) load(g, 0);
    uint32_t phase[2] = {0, 0};
    for (int i = 0; g < n_tiles; i++, g += gridDim.x) {
        const int slot = i & 1;
        const uint64_t gn = g + gridDim.x;
        if (t == 0 && gn < n_tiles) {
            // the other buffer's previous store must have read smem
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            load(gn, slot ^ 1);
        }
        // wait for this tile
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bar[slot])), "r"(phase[slot]) : "memory");
        phase[slot] ^= 1;
        // touch the data (swap re / im) so the store writes what the threads wrote
        double2 *b = buf + slot * T;
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const double2 v = b[t + u * 128];
            b[t + u * 128] = make_double2(v.y, v.x);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (t == 0) {
            int c[4];
            coords(g, c);
            asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&tm),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(smem_u32(b))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;");
        }
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int n = 26;
    const uint64_t N = 1ull << n;
    double2 *s;
    if (cudaMalloc(&s, N * 16) != cudaSuccess) return 1;
    cudaMemset(s, 0, N * 16);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (!fn) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    EncodeFn encode = (EncodeFn)fn;
    const size_t smem = 2 * T * 16;
    cudaFuncSetAttribute(sweep_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sweep_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int Cs[] = {3, 3, 3, 3, 4, 5, 11};
    const int His[] = {8, 12, 16, 18, 18, 18, 11};
    for (int pi = 0; pi < 7; pi++) {
        Shape sh{n, Cs[pi], His[pi] < Cs[pi] ? Cs[pi] : His[pi]};
        if (sh.C == K) sh.hi = K;
        const uint64_t n_tiles = N >> K;
        // tensor: d0 = 2^C amplitudes as 2 * 2^C doubles, d1 = the free bits [C, hi),
        // d2 = the tile's high block, d3 = the free bits above it
        const int gap = sh.hi - sh.C, top = n - (sh.hi + K - sh.C);
        cuuint64_t dims[4] = {(cuuint64_t)(2u << sh.C), 1ull << gap, 1ull << (K - sh.C), 1ull << top};
        cuuint64_t strides[3] = {16ull << sh.C, 16ull << sh.hi, 16ull << (sh.hi + K - sh.C)};
        cuuint32_t box[4] = {(cuuint32_t)(2u << sh.C), 1, (cuuint32_t)(1u << (K - sh.C)), 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUtensorMap tm;
        bool tma_ok = true;
        if (box[0] > 256 || box[2] > 256) tma_ok = false;   // box dims <= 256
        if (tma_ok) {
            CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, s, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("encode failed %d for C=%d hi=%d\n", (int)r, sh.C, sh.hi); tma_ok = false; }
        }
        for (int mode = 0; mode < 2; mode++) {
            if (mode == 1 && !tma_ok) continue;
            for (int occ : {3, 6}) {
                const int grid = sms * occ;
                auto launch = [&]() {
                    if (mode == 0) sweep_ldgsts<<<grid, 128, smem>>>(s, n_tiles, sh);
                    else sweep_tma<<<grid, 128, smem + 1024>>>(tm, n_tiles, sh);
                };
                launch();
                cudaEventRecord(a);
                const int R = 5;
                for (int r = 0; r < R; r++) launch();
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                cudaError_t e = cudaGetLastError();
                printf("{\"mode\": \"%s\", \"C\": %d, \"hi\": %d, \"ctas_per_sm\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n",
                       mode ? "tma" : "ldgsts", sh.C, sh.hi, occ, 32.0 * N * R / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
