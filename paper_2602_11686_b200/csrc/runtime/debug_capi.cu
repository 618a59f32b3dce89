// Test-only C entry point: runs one grouped tcgen05 GEMM on caller-provided
// device buffers so the kernel can be checked in isolation against a torch fp32
// matmul (tests/test_gpu_gemm.py).  Not used by the layer step.
#include "host/capi_common.hpp"
#include "kernels/fsep_types.cuh"
#include "kernels/kernels.hpp"
#include "moeplan_fsep.h"

extern "C" {

// b_d0/b_d1/b_groups/b_pitch1/b_pitch2 describe B: for the M-grouped kinds a 3-D
// bf16 tensor [groups][d1][d0] (pitches in elements); for the wgrad kind a 2-D
// tensor [b_d1 rows][b_d0] with pitch b_pitch1.
__attribute__((visibility("default"))) mp_status mp_fsep_debug_grouped_gemm(
    int kind, int num_groups, const int* group_rows, const int* group_off, int M, int N, int K, const void* A,
    unsigned long long a_rows, unsigned long long a_inner, unsigned long long a_pitch, const void* B,
    unsigned long long b_d0, unsigned long long b_d1, unsigned long long b_groups, unsigned long long b_pitch1,
    unsigned long long b_pitch2, void* out, long long ldo, long long out_gstride, void* out2, long long ldo2,
    const void* aux, long long ld_aux, void* stream) {
  using namespace fsep;
  return moeplan::capi::guarded([&] {
    const bool pair = (kind & 0x100) != 0;  // CTA-pair kernel (cta_group::2)
    const GemmKind k = static_cast<GemmKind>(kind & 0xf);
    const bool a_mn = k == GemmKind::kBwdWgrad;
    const bool b_mn = k != GemmKind::kFwdGateUp && k != GemmKind::kFwdDown;
    CUtensorMap ta = a_mn ? make_tmap_2d(A, a_inner, a_rows, a_pitch, 64, 64) : make_tmap_2d(A, a_inner, a_rows, a_pitch, 64, 128);
    CUtensorMap tb;
    if (k == GemmKind::kBwdWgrad)
      tb = make_tmap_2d(B, b_d0, b_d1, b_pitch1, 64, 64);
    else if (b_mn)
      tb = make_tmap_3d(B, b_d0, b_d1, b_groups, b_pitch1, b_pitch2, 64, 64);
    else
      tb = make_tmap_3d(B, b_d0, b_d1, b_groups, b_pitch1, b_pitch2, 64, pair ? 128 : 256);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    GroupedGemmArgs g{num_groups, group_rows, group_off, M, N, K, out, ldo, out_gstride, out2, ldo2, aux, ld_aux};
    // experiment knobs: bits 12-15 L2 policy, 16-23 raster, 24-27 GemmParams::policy bits 8-11
    g.policy = ((kind >> 12) & 0xF) | (((kind >> 24) & 0xF) << 8);
    g.raster = (kind >> 16) & 0xFF;
    static int* wave_sync = nullptr;  // wave-synchronisation counters, as the layer step passes them
    if (wave_sync == nullptr && cudaMalloc(&wave_sync, kWaveSyncMax * sizeof(int)) != cudaSuccess)
      throw moeplan::Error(moeplan::ErrorKind::device, "cudaMalloc(wave_sync) failed");
    g.wave_sync = wave_sync;
    CUtensorMap tb64{};
    if (pair && k == GemmKind::kFwdGateUp) {  // M=128 tail tiles stage B as [gate 64 | up 64]
      tb64 = make_tmap_3d(B, b_d0, b_d1, b_groups, b_pitch1, b_pitch2, 64, 64);
      g.b64 = &tb64;
    }
    if (pair)
      launch_grouped_gemm_pair(k, ta, tb, g, sms, static_cast<cudaStream_t>(stream));
    else
      launch_grouped_gemm(k, ta, tb, g, sms, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw moeplan::Error(moeplan::ErrorKind::device, cudaGetErrorString(e));
  });
}

// Dev builds only (-DFSEP_GEMM_STALLS via FSEP_NVCC_EXTRA): role wait-cycle totals.
__attribute__((visibility("default"))) mp_status mp_fsep_debug_gemm_stalls(unsigned long long* out8, int reset) {
  return moeplan::capi::guarded([&] {
    if (!fsep::gemm_stall_counters(out8, reset != 0))
      throw moeplan::Error(moeplan::ErrorKind::invalid_argument, "built without FSEP_GEMM_STALLS");
  });
}

}  // extern "C"
