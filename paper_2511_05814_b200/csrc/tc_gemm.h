// Host interface of the tcgen05 grouped GEMM (tc_gemm.cuh).
#pragma once
#include "tc_gemm.cuh"

namespace moe {
namespace tc {

// 2-D bf16 tensor map over a row-major [rows][cols] matrix: 64 x 128 boxes, 128-byte swizzle.
moe_status make_tmap_bf16(CUtensorMap* map, const void* base, long long rows, long long cols);
// Persistent launch (grid CTAs) of grouped_gemm_kernel.
moe_status launch_grouped(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                          const Params& p, int grid, cudaStream_t s);
int sm_count();

}  // namespace tc
}  // namespace moe
