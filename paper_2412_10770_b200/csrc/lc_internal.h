// lc_internal.h -- declarations shared by lc_host.cpp and lc_kernels.cu (product only).
#pragma once
#include <cstdint>

#include "lc.h"

namespace lc_detail {
// b = ceil(log2(2 eps + 1))
uint32_t res_bits(uint64_t eps);
// FORMAT F1/F2 header consistency (layout recomputed from n, L, b)
int32_t check_header(const lc_header* h, uint64_t blob_bytes);
// bump the kernel-launch counter reported by lc_launch_count()
void count_launch(uint64_t k);
// full-decode kernel tables, one per (kind, key width) translation unit (lc_decode_inst.cu):
// decode_kernel_<kind>_<k64>(b) = &lc_decode_kernel<k64, b, kind == 1, kind == 2>
const void* decode_kernel_0_0(uint32_t b);
const void* decode_kernel_0_1(uint32_t b);
const void* decode_kernel_1_0(uint32_t b);
const void* decode_kernel_1_1(uint32_t b);
const void* decode_kernel_2_0(uint32_t b);
const void* decode_kernel_2_1(uint32_t b);
#ifdef LC_DEBUG_BOUNDS
uint32_t debug_violations_0_0(uint32_t* where3);
uint32_t debug_violations_0_1(uint32_t* where3);
uint32_t debug_violations_1_0(uint32_t* where3);
uint32_t debug_violations_1_1(uint32_t* where3);
uint32_t debug_violations_2_0(uint32_t* where3);
uint32_t debug_violations_2_1(uint32_t* where3);
#endif
}  // namespace lc_detail
