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
}  // namespace lc_detail
