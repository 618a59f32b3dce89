// Host-side launch API of the FSEP sm_100a kernels (used by the runtime and the
// C ABI).  Every launcher is asynchronous on the given stream.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace fsep {

// ------------------------------------------------------------------ TMA maps
// 2-D bf16 tensor [outer][inner] (inner contiguous), row pitch in elements.
CUtensorMap make_tmap_2d(const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_elems, uint32_t box_inner,
                         uint32_t box_outer);
// 3-D bf16 tensor [d2][d1][d0] with explicit pitches (elements) for d1 and d2.
CUtensorMap make_tmap_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t pitch1, uint64_t pitch2,
                         uint32_t box0, uint32_t box1);

// ------------------------------------------------------------------ GEMMs
struct GroupedGemmArgs {
  int num_groups;
  const int* group_rows;  // device, padded (multiple of 128)
  const int* group_off;   // device
  int M, N, K;
  void* out;
  long long ldo;
  long long out_group_stride;
  void* out2;
  long long ldo2;
  const void* aux;
  long long ld_aux;
  int policy = 0;  // see GemmParams
  int raster = 0;
  const unsigned* ready = nullptr;  // per-group readiness flags (see GemmParams)
  unsigned ready_epoch = 0;
  int ready_n = 0;
  unsigned* err = nullptr;  // host-mapped error words (fsep_types.cuh ErrWord)
  unsigned long long ready_timeout_ns = 10000000000ull;
  const int* row_src = nullptr;  // optional row scatter of the bf16 epilogue (see GemmParams)
  __nv_bfloat16* const* scatter = nullptr;
  long long scatter_rows = 0;
  int* wave_sync = nullptr;  // optional wave-synchronisation counters (see GemmParams), zeroed by the launcher
  const CUtensorMap* b64 = nullptr;  // gate-up only: B map with 64-row boxes (M=128 tail tiles' [gate|up] staging)
};

enum class GemmKind : int {
  kFwdGateUp = 0,  // h,act = swiglu(X[rows,H] * W13_g[2F,H]^T)        A K-major, B K-major (3-D)
  kFwdDown = 1,    // Y = act[rows,F] * W2_g[H,F]^T                       A K-major, B K-major (3-D)
  kBwdDownDgrad = 2,  // dH = swiglu'(dY[rows,H] * W2_g[H,F]) using h      A K-major, B MN-major (3-D)
  kBwdUpDgrad = 3,    // dX = dH[rows,2F] * W13_g[2F,H]                   A K-major, B MN-major (3-D)
  kBwdWgrad = 4,      // dW_g = A_g^T * B_g over the group's rows (fp32)   A MN-major, B MN-major (2-D)
};

// Single-CTA 128x256 tiles (B maps with 256-row boxes for the K-major weight operand).
void launch_grouped_gemm(GemmKind kind, const CUtensorMap& tmA, const CUtensorMap& tmB, const GroupedGemmArgs& args,
                         int num_sms, cudaStream_t stream);
// CTA-pair 256x256 tiles (cta_group::2; K-major B maps with 128-row boxes).  Production path.
bool pair_gemm_supported(GemmKind kind, const GroupedGemmArgs& args);
void launch_grouped_gemm_pair(GemmKind kind, const CUtensorMap& tmA, const CUtensorMap& tmB,
                              const GroupedGemmArgs& args, int num_sms, cudaStream_t stream);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, current device):
// function attributes belong to each device's context, so a process driving several
// GPUs must set them on every device it launches on.
void set_smem_attr(const void* func, int bytes);

// Kernel-count bookkeeping for bench/roofline (launches issued by this library).
uint64_t launches_issued();
// Dev builds (-DFSEP_GEMM_STALLS): per-role barrier-wait cycle totals of the pair
// GEMM (grouped_gemm2.cuh g_gemm_stall); false when compiled out.
bool gemm_stall_counters(unsigned long long* out8, bool reset);
void count_launch(int n = 1);

}  // namespace fsep
