// Host launchers for the grouped tcgen05 GEMM (grouped_gemm.cuh) and TMA
// tensor-map construction (driver entry point fetched through the runtime, so
// the library does not link libcuda directly).
#include <cstdlib>
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>
#include <set>
#include <utility>
#include <stdexcept>
#include <string>

#include "kernels/grouped_gemm.cuh"
#include "kernels/grouped_gemm2.cuh"
#include "kernels/kernels.hpp"

namespace fsep {

namespace {
std::atomic<uint64_t> g_launches{0};

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

void check_encode(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw std::runtime_error(std::string("cuTensorMapEncodeTiled failed: ") + what);
}
}  // namespace

uint64_t launches_issued() { return g_launches.load(); }

void set_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({func, dev}).second) cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

bool gemm_stall_counters(unsigned long long* out, bool reset) {
#ifdef FSEP_GEMM_STALLS
  if (cudaMemcpyFromSymbol(out, g_gemm_stall, sizeof(g_gemm_stall)) != cudaSuccess) return false;
  if (reset) {
    const unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_gemm_stall, z, sizeof(z));
  }
  return true;
#else
  (void)out;
  (void)reset;
  return false;
#endif
}
// Every launcher calls this right after its launch: count it, and surface launch
// errors (bad configuration, shared-memory limits) at the call that caused them.
void count_launch(int n) {
  g_launches += static_cast<uint64_t>(n);
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
  }
}

CUtensorMap make_tmap_2d(const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_elems, uint32_t box_inner,
                         uint32_t box_outer) {
  CUtensorMap m{};
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {pitch_elems * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  check_encode(encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
               "2d");
  return m;
}

CUtensorMap make_tmap_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t pitch1, uint64_t pitch2,
                         uint32_t box0, uint32_t box1) {
  CUtensorMap m{};
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {pitch1 * 2, pitch2 * 2};
  const cuuint32_t box[3] = {box0, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  check_encode(encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
               "3d");
  return m;
}

namespace {
template <bool AMN, bool BMN, bool GK, int EPI>
void launch_one(const CUtensorMap& a, const CUtensorMap& b, const GemmParams& p, int grid, cudaStream_t st) {
  auto kern = grouped_gemm_kernel<AMN, BMN, GK, EPI>;
  set_smem_attr(reinterpret_cast<const void*>(kern), gemm::SMEM_BYTES);
  kern<<<grid, gemm::THREADS, gemm::SMEM_BYTES, st>>>(a, b, p);
  count_launch();
}
}  // namespace

namespace {
int env_raster(int kind) {
  const std::string name = "FSEP_MRASTER_" + std::to_string(kind);
  const char* v = std::getenv(name.c_str());
  if (!v) v = std::getenv("FSEP_MRASTER");
  return v ? std::atoi(v) : 0;
}

template <bool AMN, bool BMN, bool GK, int EPI>
void launch_pair(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& b64, const GemmParams& p, int grid,
                 cudaStream_t st) {
  auto kern = grouped_gemm_pair_kernel<AMN, BMN, GK, EPI>;
  set_smem_attr(reinterpret_cast<const void*>(kern), gemm2::smem_bytes(EPI));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid & ~1));
  cfg.blockDim = dim3(gemm2::THREADS);
  cfg.dynamicSmemBytes = gemm2::smem_bytes(EPI);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, a, b, b64, p);
  count_launch();
}
}  // namespace

bool pair_gemm_supported(GemmKind kind, const GroupedGemmArgs& a) {
  return kind != GemmKind::kBwdWgrad || a.M % gemm2::BM == 0;
}

void launch_grouped_gemm_pair(GemmKind kind, const CUtensorMap& tmA, const CUtensorMap& tmB,
                              const GroupedGemmArgs& a, int num_sms, cudaStream_t stream) {
  if (a.num_groups > gemm2::MAX_GROUPS) throw std::runtime_error("grouped gemm: too many groups");
  if (a.N % 32 != 0) throw std::runtime_error("grouped gemm: N must be a multiple of 32");
  if (!pair_gemm_supported(kind, a)) throw std::runtime_error("pair gemm: wgrad M must be a multiple of 256");
  GemmParams p{a.num_groups, a.group_rows, a.group_off, a.M,    a.N,    a.K,   a.out,
               a.ldo,        a.out_group_stride, a.out2,    a.ldo2, a.aux, a.ld_aux, a.policy, a.raster,
               a.ready,      a.ready_epoch,      a.ready_n,      a.err, a.ready_timeout_ns,
               a.row_src,    a.scatter,          a.scatter_rows, nullptr};
  static const bool wave_sync = [] {  // FSEP_WAVE_SYNC=0: free-running producers
    const char* v = std::getenv("FSEP_WAVE_SYNC");
    return !(v && std::string(v) == "0");
  }();
  // long-K M-grouped GEMMs only: their A / B panels (256 x K) do not stay in L2 when the
  // CTA pairs drift apart along K (Mixtral up-dgrad, K = 28672: DRAM reads 11.9 -> 9.7 GB,
  // step +2.5-5%); short-K panels fit in L2 anyway and the barrier only costs (fine config)
  // K-grouped wgrad: every launch.  A wave that mixes groups of different row counts idles
  // at the barrier (LPT order keeps neighbours similar), but free-running pairs drift apart
  // along the hot experts' long K and re-read their panels: fine dW13 DRAM reads 10.9 ->
  // 3.6 GB, fine step +0.6 to +3.5 % at N=1 and +1.7 % at N=4 (profiles/r02/wgrad_sync/).
  // FSEP_WAVE_SYNC_WGRAD=0: free-running; =big: only groups spanning >= 2 waves (round 1)
  static const int wave_sync_min_k = [] {  // FSEP_WAVE_SYNC_MIN_K: shortest K synchronised (A/B)
    const char* v = std::getenv("FSEP_WAVE_SYNC_MIN_K");
    return v ? std::atoi(v) : 4096;
  }();
  static const int wave_sync_wgrad = [] {
    const char* v = std::getenv("FSEP_WAVE_SYNC_WGRAD");
    return !v ? 2 : std::string(v) == "0" ? 0 : std::string(v) == "big" ? 1 : 2;
  }();
  const bool long_k =
      kind == GemmKind::kBwdWgrad
          ? wave_sync_wgrad == 2 ||
                (wave_sync_wgrad == 1 && (a.M / gemm2::BM) * ((a.N + gemm2::BN - 1) / gemm2::BN) >= 2 * num_sms)
          : a.K >= wave_sync_min_k;
  // Tile order of the wgrad launches: for groups spanning several waves, the panels along
  // the shorter tile dimension stay resident in L2 for the whole group while the other side
  // streams past them once -- n fastest when a group has no more n tiles than m tiles
  // (Mixtral dW13, 112 x 16: DRAM reads 6.3 -> 4.4 GB, step +0.5 %), else 16-tile m-chunks
  // (dW2, 16 x 56: n-fastest there would re-read 8 GB; small groups, e.g. the fine
  // config's 11 x 8, measured level-to-worse with n-fastest).  FSEP_WGRAD_RASTER overrides.
  static const int wgrad_raster = [] {
    const char* v = std::getenv("FSEP_WGRAD_RASTER");
    return v ? std::atoi(v) : -1;
  }();
  if (kind == GemmKind::kBwdWgrad && p.raster == 0) {
    const int m_tiles = a.M / gemm2::BM, n_tiles = (a.N + gemm2::BN - 1) / gemm2::BN;
    const bool big = m_tiles * n_tiles >= 2 * num_sms;
    p.raster = wgrad_raster >= 0 ? wgrad_raster : (big && n_tiles <= m_tiles ? 2 : 0);
  }
  // FSEP_MRASTER[_<kind>]: m-chunk of the M-grouped launches' tile order (A/B; default 16 m tiles,
  // n-inner: an A chunk of 16 x 256 rows stays in L2 while the B panels stream past it)
  static const int mraster[4] = {env_raster(0), env_raster(1), env_raster(2), env_raster(3)};
  if (kind != GemmKind::kBwdWgrad && p.raster == 0) p.raster = mraster[static_cast<int>(kind)];
  static const int wave_kinds = [] {  // FSEP_WAVE_SYNC_KINDS: bit k = wave sync allowed for GemmKind k (A/B)
    const char* v = std::getenv("FSEP_WAVE_SYNC_KINDS");
    return v ? static_cast<int>(std::strtol(v, nullptr, 0)) : 0x1F;
  }();
  if (wave_sync && a.wave_sync != nullptr && long_k && !(a.policy & 0x800) &&
      ((wave_kinds >> static_cast<int>(kind)) & 1)) {  // policy bit 11: A/B off
    cudaMemsetAsync(a.wave_sync, 0, kWaveSyncMax * sizeof(int), stream);
    p.wave_sync = a.wave_sync;
  }
  static const bool no_tail = [] {
    const char* v = std::getenv("FSEP_GEMM_NTAIL");
    return v && std::string(v) == "0";
  }();
  if (no_tail) p.policy |= 0x100;
  static const bool rr_sched = [] {  // FSEP_GEMM_SCHED=rr: plain round robin, groups in index order
    const char* v = std::getenv("FSEP_GEMM_SCHED");
    return v && std::string(v) == "rr";
  }();
  if (rr_sched) p.policy |= 0x200;
  static const bool rel_cluster = [] {  // FSEP_TMEM_RELEASE=cluster: cluster-scope release on the TMEM hand-off
    const char* v = std::getenv("FSEP_TMEM_RELEASE");
    return v && std::string(v) == "cluster";
  }();
  if (rel_cluster) p.policy |= 0x400;
  static const bool no_mtail = [] {  // FSEP_GEMM_MTAIL=0: masked M=256 tail tiles (A/B)
    const char* v = std::getenv("FSEP_GEMM_MTAIL");
    return v && std::string(v) == "0";
  }();
  if (no_mtail) p.policy |= 0x1000;
  // FSEP_KSNAKE: bit k = odd waves of GemmKind k load K backwards.  Default: every kind but
  // the gate-up GEMM (measured: -7 to -19 % DRAM reads on the other launches, Mixtral
  // step +1.2 %, fine level; gate-up reads +2 %)
  static const int ksnake_kinds = [] {
    const char* v = std::getenv("FSEP_KSNAKE");
    return v ? static_cast<int>(std::strtol(v, nullptr, 0)) : 0x1E;
  }();
  if ((ksnake_kinds >> static_cast<int>(kind)) & 1) p.policy |= 0x4000;
  static const bool no_h_prefetch = [] {  // FSEP_H_PREFETCH=0: no L2 prefetch of h in the SwiGLU' epilogue (A/B)
    const char* v = std::getenv("FSEP_H_PREFETCH");
    return v && std::string(v) == "0";
  }();
  if (no_h_prefetch) p.policy |= 0x8000;
  // the gate-up GEMM's M=128 tail tiles stage B as [gate 64 | up 64] halves (64-row box map)
  const CUtensorMap& b64 = a.b64 != nullptr ? *a.b64 : tmB;
  if (kind == GemmKind::kFwdGateUp && a.b64 != nullptr) p.policy |= 0x2000;
  switch (kind) {
    case GemmKind::kFwdGateUp: launch_pair<false, false, false, kEpiSwigluFwd>(tmA, tmB, b64, p, num_sms, stream); break;
    case GemmKind::kFwdDown: launch_pair<false, false, false, kEpiBf16>(tmA, tmB, b64, p, num_sms, stream); break;
    case GemmKind::kBwdDownDgrad: launch_pair<false, true, false, kEpiSwigluBwd>(tmA, tmB, b64, p, num_sms, stream); break;
    case GemmKind::kBwdUpDgrad: launch_pair<false, true, false, kEpiBf16>(tmA, tmB, b64, p, num_sms, stream); break;
    case GemmKind::kBwdWgrad: launch_pair<true, true, true, kEpiF32>(tmA, tmB, b64, p, num_sms, stream); break;
  }
}

void launch_grouped_gemm(GemmKind kind, const CUtensorMap& tmA, const CUtensorMap& tmB, const GroupedGemmArgs& a,
                         int num_sms, cudaStream_t stream) {
  if (a.num_groups > gemm::MAX_GROUPS) throw std::runtime_error("grouped gemm: too many groups");
  if (a.N % 32 != 0) throw std::runtime_error("grouped gemm: N must be a multiple of 32");
  GemmParams p{a.num_groups, a.group_rows, a.group_off, a.M,    a.N,    a.K,   a.out,
               a.ldo,        a.out_group_stride, a.out2,    a.ldo2, a.aux, a.ld_aux, a.policy, a.raster,
               a.ready,      a.ready_epoch,      a.ready_n,      a.err, a.ready_timeout_ns,
               a.row_src,    a.scatter,          a.scatter_rows, nullptr};
  switch (kind) {
    case GemmKind::kFwdGateUp: launch_one<false, false, false, kEpiSwigluFwd>(tmA, tmB, p, num_sms, stream); break;
    case GemmKind::kFwdDown: launch_one<false, false, false, kEpiBf16>(tmA, tmB, p, num_sms, stream); break;
    case GemmKind::kBwdDownDgrad: launch_one<false, true, false, kEpiSwigluBwd>(tmA, tmB, p, num_sms, stream); break;
    case GemmKind::kBwdUpDgrad: launch_one<false, true, false, kEpiBf16>(tmA, tmB, p, num_sms, stream); break;
    case GemmKind::kBwdWgrad: launch_one<true, true, true, kEpiF32>(tmA, tmB, p, num_sms, stream); break;
  }
}

}  // namespace fsep
