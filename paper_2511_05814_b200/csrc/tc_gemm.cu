// Host side of the tcgen05 grouped GEMM (K4): tensor-map construction and the test /
// microbenchmark entry points.  The prefill path (prefill.cu) launches the same kernel with
// device-prepared tile tables.
#define MOE_TC_GEMM_KERNEL
#include "tc_gemm.h"

#include <mutex>
#include <vector>

namespace moe {
namespace tc {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}
}  // namespace

moe_status make_tmap_bf16(CUtensorMap* map, const void* base, long long rows, long long cols) {
  EncodeFn fn = encode_fn();
  MOE_REQUIRE(fn, "cuTensorMapEncodeTiled is not available from the driver");
  MOE_REQUIRE(cols % BK == 0 && rows >= 1, "tensor map needs cols %% 64 == 0 (got %lld x %lld)", rows, cols);
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  const cuuint32_t box[2] = {BK, 128};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for %lld x %lld at %p", static_cast<int>(r), rows,
              cols, base);
    return MOE_CUDA_ERROR;
  }
  return MOE_OK;
}

moe_status launch_grouped(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                          const Params& p, int grid, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(grouped_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  });
  grouped_gemm_kernel<<<grid, THREADS, SMEM_BYTES, s>>>(a, b0, b1, p);
  MOE_LAUNCHED();
  return MOE_OK;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace tc
}  // namespace moe

using namespace moe;

namespace {
// Host-built tile table for the test entry points: groups contiguous in A, n-tiles outer,
// m-tiles inner (the m-tiles sharing a weight tile run side by side and share it in L2).
struct HostPlan {
  std::vector<tc::Group> groups;
  std::vector<tc::Tile> tiles;
};

HostPlan plan_groups(int G, const int32_t* group_m, int N_tile_cols, int n_cols, int b_rows_per_group,
                     bool swiglu, int f) {
  HostPlan hp;
  int row = 0;
  for (int g = 0; g < G; ++g) {
    tc::Group gr{};
    gr.a_row0 = row;
    gr.m = group_m[g];
    gr.b_row0 = g * b_rows_per_group;
    gr.b_row1 = swiglu ? gr.b_row0 + f : 0;
    hp.groups.push_back(gr);
    for (int n0 = 0; n0 < n_cols; n0 += N_tile_cols)
      for (int m0 = 0; m0 < gr.m; m0 += tc::BM) hp.tiles.push_back(tc::Tile{g, m0, n0});
    row += gr.m;
  }
  return hp;
}

moe_status run_plan(const HostPlan& hp, const CUtensorMap& ta, const CUtensorMap& tb, tc::Params p,
                    int grid, int iters, cudaStream_t s, float* ms) {
  void* dev = nullptr;
  const size_t gbytes = sizeof(tc::Group) * hp.groups.size();
  const size_t tbytes = sizeof(tc::Tile) * std::max<size_t>(1, hp.tiles.size());
  MOE_CUDA(cudaMalloc(&dev, gbytes + tbytes + 16));
  char* base = static_cast<char*>(dev);
  MOE_CUDA(cudaMemcpyAsync(base, hp.groups.data(), gbytes, cudaMemcpyHostToDevice, s));
  if (!hp.tiles.empty())
    MOE_CUDA(cudaMemcpyAsync(base + gbytes, hp.tiles.data(), sizeof(tc::Tile) * hp.tiles.size(),
                             cudaMemcpyHostToDevice, s));
  const int nt = static_cast<int>(hp.tiles.size());
  MOE_CUDA(cudaMemcpyAsync(base + gbytes + tbytes, &nt, sizeof(int), cudaMemcpyHostToDevice, s));
  p.groups = reinterpret_cast<const tc::Group*>(base);
  p.tiles = reinterpret_cast<const tc::Tile*>(base + gbytes);
  p.n_tiles = reinterpret_cast<const int*>(base + gbytes + tbytes);
  if (grid <= 0) grid = std::max(1, std::min(nt * std::max(1, p.splits), tc::sm_count()));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    MOE_CUDA(cudaEventCreate(&e0));
    MOE_CUDA(cudaEventCreate(&e1));
  }
  moe_status st = MOE_OK;
  for (int i = 0; i < iters && st == MOE_OK; ++i) {
    if (ms && i == (iters > 1 ? 1 : 0)) cudaEventRecord(e0, s);
    st = tc::launch_grouped(ta, tb, tb, p, grid, s);
  }
  if (ms) {
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    *ms = t / std::max(1, iters > 1 ? iters - 1 : 1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  cudaStreamSynchronize(s);
  cudaFree(dev);
  if (st != MOE_OK) return st;
  MOE_CUDA(cudaGetLastError());
  return MOE_OK;
}
}  // namespace

extern "C" {

moe_status moe_tc_grouped_gemm_bf16(const uint16_t* A, const uint16_t* B, float* C, int32_t G,
                                    const int32_t* group_m, int32_t N, int32_t K, int32_t splits,
                                    int32_t iters, float* ms_per_iter, void* stream) {
  MOE_REQUIRE(A && B && C && group_m && G >= 1, "null argument");
  MOE_REQUIRE(K % tc::BK == 0 && K >= tc::BK, "K must be a positive multiple of 64, got %d", K);
  MOE_REQUIRE(N % tc::BN == 0 && N >= tc::BN, "N must be a positive multiple of 256, got %d", N);
  MOE_REQUIRE(splits >= 1 && splits <= K / tc::BK, "splits must be in [1, K/64], got %d", splits);
  long long rows = 0;
  for (int g = 0; g < G; ++g) {
    MOE_REQUIRE(group_m[g] >= 0, "negative group size");
    rows += group_m[g];
  }
  MOE_REQUIRE(rows >= 1, "empty problem");
  cudaStream_t s = as_stream(stream);
  CUtensorMap ta, tb;
  moe_status st = tc::make_tmap_bf16(&ta, A, rows, K);
  if (st != MOE_OK) return st;
  st = tc::make_tmap_bf16(&tb, B, static_cast<long long>(G) * N, K);
  if (st != MOE_OK) return st;
  HostPlan hp = plan_groups(G, group_m, tc::BN, N, N, false, 0);
  tc::Params p{};
  p.K = K;
  p.N = N;
  p.epi = tc::kEpiStoreF32;
  p.c = C;
  p.splits = splits;
  p.split_stride = rows * N;
  return run_plan(hp, ta, tb, p, 0, std::max(1, iters), s, ms_per_iter);
}

moe_status moe_tc_grouped_swiglu_bf16(const uint16_t* X, const uint16_t* W13, uint16_t* act,
                                      int32_t G, const int32_t* group_m, int32_t f, int32_t d,
                                      int32_t iters, float* ms_per_iter, void* stream) {
  MOE_REQUIRE(X && W13 && act && group_m && G >= 1, "null argument");
  MOE_REQUIRE(d % tc::BK == 0 && d >= tc::BK, "d must be a positive multiple of 64, got %d", d);
  MOE_REQUIRE(f % (tc::BN / 2) == 0 && f >= tc::BN / 2, "f must be a positive multiple of 128, got %d", f);
  long long rows = 0;
  for (int g = 0; g < G; ++g) {
    MOE_REQUIRE(group_m[g] >= 0, "negative group size");
    rows += group_m[g];
  }
  MOE_REQUIRE(rows >= 1, "empty problem");
  cudaStream_t s = as_stream(stream);
  CUtensorMap ta, tb;
  moe_status st = tc::make_tmap_bf16(&ta, X, rows, d);
  if (st != MOE_OK) return st;
  st = tc::make_tmap_bf16(&tb, W13, static_cast<long long>(G) * 2 * f, d);
  if (st != MOE_OK) return st;
  HostPlan hp = plan_groups(G, group_m, tc::BN / 2, f, 2 * f, true, f);
  tc::Params p{};
  p.K = d;
  p.N = f;
  p.epi = tc::kEpiSwiGLU;
  p.act = act;
  return run_plan(hp, ta, tb, p, 0, std::max(1, iters), s, ms_per_iter);
}

}  // extern "C"
