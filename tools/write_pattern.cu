// tools/write_pattern.cu -- microbenchmark of HBM write patterns relevant to the decode kernel's
// output stream (each warp owns consecutive 1024-key / 8 KB chunks).  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/write_pattern tools/write_pattern.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                             \
        }                                                                         \
    } while (0)

constexpr int kWarps = 8;

// P1: grid-stride 16-byte stores (like a fill)
__global__ void p_fill(uint4* out, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = make_uint4(1, 2, 3, 4);
}

// P2/P3/P4: persistent warps, chunk c = 8 KB, 256 B (v2) or 512 B (v4) per warp store
template <int MODE>
__global__ void __launch_bounds__(256) p_chunk(uint8_t* out, uint32_t nchunks) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * kWarps;
    for (uint32_t c = blockIdx.x * kWarps + (threadIdx.x >> 5); c < nchunks; c += nw) {
        uint8_t* base = out + (size_t)c * 8192;
        if (MODE == 0) {  // st.global.cs.u64, 32 stores of 256 B
#pragma unroll 8
            for (int k = 0; k < 32; ++k)
                __stcs((unsigned long long*)(base + k * 256) + lane, (unsigned long long)c);
        } else if (MODE == 1) {  // plain st.global.u64
#pragma unroll 8
            for (int k = 0; k < 32; ++k)
                ((unsigned long long*)(base + k * 256))[lane] = (unsigned long long)c;
        } else if (MODE == 2) {  // st.global.cs.v4 (512 B per warp store)
#pragma unroll 8
            for (int k = 0; k < 16; ++k)
                __stcs((uint4*)(base + k * 512) + lane, make_uint4(c, c, c, c));
        } else {  // plain v4
#pragma unroll 8
            for (int k = 0; k < 16; ++k)
                ((uint4*)(base + k * 512))[lane] = make_uint4(c, c, c, c);
        }
    }
}

// P5: persistent warps, chunk written to smem then TMA bulk store S2G (SEG bytes per store)
template <int SEG>
__global__ void __launch_bounds__(256) p_bulk(uint8_t* out, uint32_t nchunks) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* buf = smem + warp * 2 * SEG;  // two buffers of SEG bytes
    const uint32_t nw = gridDim.x * kWarps;
    uint32_t it = 0;
    for (uint32_t c = blockIdx.x * kWarps + warp; c < nchunks; c += nw) {
        for (uint32_t part = 0; part < 8192 / SEG; ++part, ++it) {
            uint8_t* b = buf + (it & 1) * SEG;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            for (uint32_t k = lane; k < SEG / 8; k += 32) ((unsigned long long*)b)[k] = c;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 out + (size_t)c * 8192 + part * SEG),
                             "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(SEG)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// Mixed read+write per warp chunk (the decode's traffic shape without its math): read three
// slices (R0, R1, R2 bytes from three arrays) into smem with bulk copies, then write 8 KB.
// DB: double-buffer the reads (issue chunk c+nw's copies before writing chunk c).
__device__ __forceinline__ void mb_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t ph) {
    uint32_t done = 0;
    do {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done)
                     : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(ph)
                     : "memory");
    } while (!done);
}

template <bool DB, bool BULKST>
__global__ void __launch_bounds__(256) p_mixed(const uint8_t* r0, const uint8_t* r1,
                                               const uint8_t* r2, uint32_t R0, uint32_t R1,
                                               uint32_t R2, uint8_t* out, uint32_t nchunks) {
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t pagesz = (R0 + R1 + R2 + 127) & ~127u;
    const uint32_t per = 16 + (DB ? 2 : 1) * pagesz + (BULKST ? 8192 : 0);
    uint8_t* base = smem + warp * ((per + 127) & ~127u);
    uint64_t* bar = (uint64_t*)base;  // bar[0], bar[1]
    uint8_t* page[2] = {base + 16, base + 16 + pagesz};
    uint8_t* obuf = base + 16 + (DB ? 2 : 1) * pagesz;
    if (lane == 0) { mb_init(bar); mb_init(bar + 1); }
    __syncwarp();
    uint32_t ph[2] = {0, 0};
    const uint32_t nw = gridDim.x * kWarps;
    uint32_t c = blockIdx.x * kWarps + warp;
    auto issue = [&](uint32_t cc, int slot) {
        if (lane == 0) {
            mb_expect(bar + slot, R0 + R1 + R2);
            g2s(page[slot], r0 + (size_t)cc * R0, R0, bar + slot);
            g2s(page[slot] + R0, r1 + (size_t)cc * R1, R1, bar + slot);
            g2s(page[slot] + R0 + R1, r2 + (size_t)cc * R2, R2, bar + slot);
        }
    };
    if (DB && c < nchunks) issue(c, 0);
    uint32_t it = 0;
    for (; c < nchunks; c += nw, ++it) {
        const int slot = DB ? (it & 1) : 0;
        if (!DB) { __syncwarp(); issue(c, 0); }
        else if (c + nw < nchunks) { __syncwarp(); issue(c + nw, slot ^ 1); }
        mb_wait(bar + slot, ph[slot]);
        ph[slot] ^= 1;
        const uint32_t v = ((const uint32_t*)page[slot])[lane];
        uint8_t* o = out + (size_t)c * 8192;
        if (!BULKST) {
#pragma unroll 8
            for (int k = 0; k < 32; ++k) __stcs((unsigned long long*)(o + k * 256) + lane, (unsigned long long)v);
        } else {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll 8
            for (int k = 0; k < 32; ++k) ((unsigned long long*)(obuf + k * 256))[lane] = v;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o),
                             "r"((uint32_t)__cvta_generic_to_shared(obuf)), "r"(8192)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (BULKST && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// Streaming read:write mix: each thread reads 16 B from src and writes R x 16 B to dst
// (grid-stride, contiguous streams) -- the decode's ~1:3 byte ratio without its structure.
template <int R>
__global__ void p_ratio(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t nsrc) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nsrc;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(src + i);
#pragma unroll
        for (int r = 0; r < R; ++r) __stcs(dst + (size_t)r * nsrc + i, v);
    }
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t bytes = 4ull << 30;
    uint8_t* out;
    CK(cudaMalloc(&out, bytes));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t nchunks = (uint32_t)(bytes / 8192);
    auto gbs = [&](float ms) { return bytes / (ms * 1e-3) / 1e9; };
    printf("{");
    printf("\"fill_v4\": %.1f", gbs(timeit([&] { p_fill<<<sms * 8, 256>>>((uint4*)out, bytes / 16); })));
    for (int occ : {4, 6, 8}) {
        printf(", \"chunk_cs_v2_occ%d\": %.1f", occ,
               gbs(timeit([&] { p_chunk<0><<<sms * occ, 256>>>(out, nchunks); })));
        printf(", \"chunk_plain_v2_occ%d\": %.1f", occ,
               gbs(timeit([&] { p_chunk<1><<<sms * occ, 256>>>(out, nchunks); })));
        printf(", \"chunk_cs_v4_occ%d\": %.1f", occ,
               gbs(timeit([&] { p_chunk<2><<<sms * occ, 256>>>(out, nchunks); })));
        printf(", \"chunk_plain_v4_occ%d\": %.1f", occ,
               gbs(timeit([&] { p_chunk<3><<<sms * occ, 256>>>(out, nchunks); })));
    }
    for (int occ : {2, 3, 4}) {
        CK(cudaFuncSetAttribute(p_bulk<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192));
        CK(cudaFuncSetAttribute(p_bulk<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096));
        CK(cudaFuncSetAttribute(p_bulk<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2048));
        printf(", \"bulk4k_occ%d\": %.1f", occ,
               gbs(timeit([&] { p_bulk<4096><<<sms * occ, 256, 8 * 8192>>>(out, nchunks); })));
        printf(", \"bulk2k_occ%d\": %.1f", occ,
               gbs(timeit([&] { p_bulk<2048><<<sms * occ, 256, 8 * 4096>>>(out, nchunks); })));
        printf(", \"bulk1k_occ%d\": %.1f", occ,
               gbs(timeit([&] { p_bulk<1024><<<sms * occ, 256, 8 * 2048>>>(out, nchunks); })));
    }

    // mixed: config-2-like slices per 1024-key chunk: 400 B starts, 1520 B params, 1024 B words
    // (and the same bytes as one contiguous slice, and config-4-like: 48 B + 48 B + 768 B)
    for (int variant = 0; variant < 3; ++variant) {
        const uint32_t R0 = variant == 0 ? 400 : variant == 1 ? 2944 : 48;
        const uint32_t R1 = variant == 0 ? 1520 : variant == 1 ? 16 : 48;
        const uint32_t R2 = variant == 0 ? 1024 : variant == 1 ? 16 : 768;
        printf(", \"variant%d\": %d", variant, R0 + R1 + R2);
        uint8_t *a0, *a1, *a2, *o2;
        const uint32_t nc = 488281;  // config 4's chunk count (4 GB of output)
        CK(cudaMalloc(&a0, (size_t)nc * R0));
        CK(cudaMalloc(&a1, (size_t)nc * R1));
        CK(cudaMalloc(&a2, (size_t)nc * R2));
        CK(cudaMalloc(&o2, (size_t)nc * 8192));
        const double mb = (double)nc * (R0 + R1 + R2 + 8192);
        auto g2 = [&](float ms) { return mb / (ms * 1e-3) / 1e9; };
        const int pg = (R0 + R1 + R2 + 127) & ~127;
        // occ 1..3: the offered-load side of the curve (late round 2: single-buffered staging at
        // 2 CTAs per SM beats every fuller configuration on the real decode kernel)
        for (int occ : {1, 2, 3, 4, 8}) {
            int s1 = 8 * ((16 + pg + 127) & ~127), s2 = 8 * ((16 + 2 * pg + 127) & ~127);
            int s3 = 8 * ((16 + pg + 8192 + 127) & ~127), s4 = 8 * ((16 + 2 * pg + 8192 + 127) & ~127);
            CK(cudaFuncSetAttribute(p_mixed<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
            CK(cudaFuncSetAttribute(p_mixed<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
            CK(cudaFuncSetAttribute(p_mixed<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s3));
            CK(cudaFuncSetAttribute(p_mixed<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s4));
            int o1 = 0, o2b = 0, o3 = 0, o4 = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, p_mixed<false, false>, 256, s1);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2b, p_mixed<true, false>, 256, s2);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, p_mixed<false, true>, 256, s3);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o4, p_mixed<true, true>, 256, s4);
            printf(", \"mixed_sb_stg_occ%d(max%d)\": %.1f", occ, o1,
                   g2(timeit([&] { p_mixed<false, false><<<sms * (occ < o1 ? occ : o1), 256, s1>>>(a0, a1, a2, R0, R1, R2, o2, nc); })));
            printf(", \"mixed_db_stg_occ%d(max%d)\": %.1f", occ, o2b,
                   g2(timeit([&] { p_mixed<true, false><<<sms * (occ < o2b ? occ : o2b), 256, s2>>>(a0, a1, a2, R0, R1, R2, o2, nc); })));
            printf(", \"mixed_sb_bulk_occ%d(max%d)\": %.1f", occ, o3,
                   g2(timeit([&] { p_mixed<false, true><<<sms * (occ < o3 ? occ : o3), 256, s3>>>(a0, a1, a2, R0, R1, R2, o2, nc); })));
            printf(", \"mixed_db_bulk_occ%d(max%d)\": %.1f", occ, o4,
                   g2(timeit([&] { p_mixed<true, true><<<sms * (occ < o4 ? occ : o4), 256, s4>>>(a0, a1, a2, R0, R1, R2, o2, nc); })));
        }
        CK(cudaGetLastError());
        cudaFree(a0); cudaFree(a1); cudaFree(a2); cudaFree(o2);
    }

    {   // streaming ratio mixes: read 1 GB, write R GB
        const size_t ns = (1ull << 30) / 16;
        uint4 *src, *dst;
        CK(cudaMalloc(&src, ns * 16));
        CK(cudaMalloc(&dst, 4 * ns * 16));
        cudaMemset(src, 1, ns * 16);
        auto gb = [&](float ms, int r) { return (1.0 + r) * ns * 16 / (ms * 1e-3) / 1e9; };
        for (int g : {4, 8, 16}) {
            printf(", \"ratio1_1_g%d\": %.1f", g, gb(timeit([&] { p_ratio<1><<<sms * g, 256>>>(src, dst, ns); }), 1));
            printf(", \"ratio1_2_g%d\": %.1f", g, gb(timeit([&] { p_ratio<2><<<sms * g, 256>>>(src, dst, ns); }), 2));
            printf(", \"ratio1_3_g%d\": %.1f", g, gb(timeit([&] { p_ratio<3><<<sms * g, 256>>>(src, dst, ns); }), 3));
            printf(", \"ratio1_4_g%d\": %.1f", g, gb(timeit([&] { p_ratio<4><<<sms * g, 256>>>(src, dst, ns); }), 4));
        }
        cudaFree(src); cudaFree(dst);
    }
    CK(cudaGetLastError());
    printf("}\n");
    return 0;
}
