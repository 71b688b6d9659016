// lc_decode_inst.cu -- one set of full-decode kernel instantiations (lc_decode_kernel for every
// residual width b = 0..32) for one (kind, key width), compiled once per set with
//   -DLC_INST_KIND=0|1|2 (dense | sparse | lc_union's shifted decode) -DLC_INST_K64=0|1
// so the 198 decode kernels build in parallel translation units (_build.py).  The launcher in
// lc_kernels.cu fetches the kernel pointers through lc_detail::decode_kernel_<kind>_<k64>.
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <utility>

#include "lc.h"
#include "lc_internal.h"

#ifndef LC_INST_KIND
#error "compile with -DLC_INST_KIND=0|1|2 -DLC_INST_K64=0|1"
#endif

namespace {
#include "lc_common.cuh"
#include "lc_decode.cuh"

constexpr bool kSparse = LC_INST_KIND == 1;
constexpr bool kUni = LC_INST_KIND == 2;
constexpr bool kK64 = LC_INST_K64 != 0;

template <uint32_t... Bs>
constexpr std::array<const void*, sizeof...(Bs)> table(std::integer_sequence<uint32_t, Bs...>) {
    return {{(const void*)&lc_decode_kernel<kK64, Bs, kSparse, kUni>...}};
}
const std::array<const void*, 33> kTable = table(std::make_integer_sequence<uint32_t, 33>{});
}  // namespace

#define LC_CAT2(a, b, c) a##_##b##_##c
#define LC_CAT(a, b, c) LC_CAT2(a, b, c)

namespace lc_detail {
const void* LC_CAT(decode_kernel, LC_INST_KIND, LC_INST_K64)(uint32_t b) {
    return b < 33 ? kTable[b] : nullptr;
}
#ifdef LC_DEBUG_BOUNDS
uint32_t LC_CAT(debug_violations, LC_INST_KIND, LC_INST_K64)(uint32_t* where3) {
    return debug_take(where3);
}
#endif
}  // namespace lc_detail
