// tools/gather_pattern.cu -- DRAM cost of random 16-byte gathers (the access kernel's params
// load) under different load flavours.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_pattern tools/gather_pattern.cu
//   ncu --metrics dram__sectors_read.sum,gpu__time_duration.sum ./build/gather_pattern
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#ifndef NSRC
#define NSRC 7500000ull
#endif

template <int MODE>
__global__ void __launch_bounds__(256) gather(const ulonglong2* __restrict__ src,
                                              const uint32_t* __restrict__ idx, uint64_t q,
                                              unsigned long long* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (t >= q) return;
    const uint32_t i = __ldcs(idx + t);
    ulonglong2 v;
    if (MODE == 0) {
        v = __ldg(src + i);
    } else if (MODE == 1) {
        asm volatile("ld.global.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(src + i));
    } else if (MODE == 2) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];"
                     : "=l"(v.x), "=l"(v.y)
                     : "l"(src + i));
    } else if (MODE == 3) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                     : "=l"(v.x), "=l"(v.y)
                     : "l"(src + i), "l"(pol));
    } else if (MODE == 4) {
        asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(src + i));
    } else if (MODE == 5) {
        asm volatile("ld.global.cs.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(src + i));
    } else {
        asm volatile("ld.global.lu.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(src + i));
    }
    __stcs(out + t, v.x ^ v.y);
}

// baseline: sequential 16-byte reads (no randomness)
__global__ void seq(const ulonglong2* __restrict__ src, uint64_t q, unsigned long long* out) {
    const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (t >= q) return;
    const ulonglong2 v = __ldg(src + t);
    __stcs(out + t, v.x ^ v.y);
}

int main() {
    const uint64_t nsrc = NSRC, q = 100000000;  // params-like source (NSRC x 16 B)
    ulonglong2* src;
    uint32_t* idx;
    unsigned long long* out;
    cudaMalloc(&src, nsrc * 16);
    cudaMalloc(&idx, q * 4);
    cudaMalloc(&out, q * 8);
    cudaMemset(src, 1, nsrc * 16);
    uint32_t* h = new uint32_t[q];
    uint64_t x = 88172645463325252ull;
    for (uint64_t t = 0; t < q; ++t) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[t] = (uint32_t)(x % nsrc);
    }
    cudaMemcpy(idx, h, q * 4, cudaMemcpyHostToDevice);
    delete[] h;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const unsigned grid = (unsigned)((q + 255) / 256);
    auto run = [&](const char* name, auto launch) {
        for (int r = 0; r < 2; ++r) launch();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%s %.3f ms %.3e gathers/s\n", name, ms, q / (ms * 1e-3));
    };
    {
        size_t g = 0;
        cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
        printf("default MaxL2FetchGranularity %zu\n", g);
        for (size_t want : {32, 64, 128}) {
            cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, want);
            cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
            char name[64];
            snprintf(name, sizeof name, "ldg_l2fetch%zu(got %zu)", want, g);
            run(name, [&] { gather<0><<<grid, 256>>>(src, idx, q, out); });
        }
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 64);
    }
    run("ldg", [&] { gather<0><<<grid, 256>>>(src, idx, q, out); });
    run("ld_plain", [&] { gather<1><<<grid, 256>>>(src, idx, q, out); });
    run("ld_nc_l1noalloc", [&] { gather<2><<<grid, 256>>>(src, idx, q, out); });
    run("ld_nc_evict_first", [&] { gather<3><<<grid, 256>>>(src, idx, q, out); });
    run("ld_cg", [&] { gather<4><<<grid, 256>>>(src, idx, q, out); });
    run("ld_cs", [&] { gather<5><<<grid, 256>>>(src, idx, q, out); });
    run("ld_lu", [&] { gather<6><<<grid, 256>>>(src, idx, q, out); });
    run("seq", [&] { seq<<<(unsigned)((nsrc + 255) / 256), 256>>>(src, nsrc, out); });
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
