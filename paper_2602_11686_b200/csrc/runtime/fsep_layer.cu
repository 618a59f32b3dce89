// FsepLayer: the B200 runtime of one FSEP MoE layer step, behind the
// mp_fsep_layer_* C ABI (include/moeplan_fsep.h).
//
// Step schedule (per rank; in virtual mode every phase loops over the N
// emulated ranks on one GPU, in real mode a peer barrier kernel separates phases):
//   forward   layout H2D | == barrier == | shard restore: every rank PUSHES its
//             chunk of each expert to the ranks hosting it (copy engines, one
//             stream per destination), each copy followed by a readiness flag
//             written into the destination's memory (virtual mode: a restore
//             kernel on a side stream)
//             router+top-k+histogram -> block scan (R row -> every rank's R_all)
//             == barrier ==  plan (device lite routing) + pad zeroing
//             R D2H + host planner callback (planner stream) -> layout of step t+1
//             dispatch (token rows -> destination rows, peer stores)
//             == barrier ==  GEMM gate/up + SwiGLU -> GEMM down (producer waits per
//             slot for its restored chunks, so the restore overlaps the GEMMs; the
//             down GEMM's epilogue stores y rows into the token owners' slot rows)
//             == barrier ==  combine (local slot rows, gate-weighted fp32 sum)
//   backward  combine bwd (dw, dl; dY rows -> expert devices) + router wgrad GEMM
//             == barrier ==  dgrad (SwiGLU'), wgrad dW13 -> push W13 grad chunks to
//             their owners (copy engines) under the dW2 wgrad and the dX GEMM ->
//             push W2 chunks under the dX GEMM (its epilogue stores dX rows into the
//             owners' slot rows)
//             == barrier ==  owner-side reduce-scatter sum, unpermute bwd (+ router dx)
// Only the copy-engine path needs the layout on the host: the forward waits on
// the previous step's planner callback (which ran right after that step's
// router), so the host stays one step ahead.  Per-expert row counts never leave
// the device (the grouped GEMMs schedule their tiles from them).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "host/capi_common.hpp"
#include "kernels/kernels.hpp"
#include "kernels/routing.hpp"
#include "moeplan/planner.hpp"
#include "moeplan_fsep.h"

using moeplan::Error;
using moeplan::ErrorKind;

namespace fsep {
namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(ErrorKind::device, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Memory guards (the memcheck stand-in: compute-sanitizer is closed on the GPU pool):
// every carved buffer is followed by kGuardBytes of 0xA5; mp_fsep_layer_check verifies
// them on the device, so a kernel writing past any buffer's end fails the step loudly.
constexpr size_t kGuardBytes = 256;
constexpr unsigned char kGuardByte = 0xA5;

struct Guard {
  const unsigned char* at;
  const char* after;  // the buffer it follows
};

struct Carver {
  char* base;
  std::vector<Guard>* guards;
  size_t off = 0;
  template <typename T>
  T* take(size_t count, const char* name) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    guards->push_back({reinterpret_cast<const unsigned char*>(base + off), name});
    off += kGuardBytes;
    return p;
  }
};

struct Rank {
  int rank = 0;
  // peer-visible arena
  void* arena = nullptr;
  size_t arena_bytes = 0;
  __nv_bfloat16 *x_rows = nullptr, *dy_rows = nullptr, *tok_rows = nullptr;
  int* row_src = nullptr;
  __nv_bfloat16* stage = nullptr;  // de-duplication: [N][T_max][H] token rows from each source
  float* row_w = nullptr;          // de-duplication: [cap] w_k of each receive row
  unsigned long long* R_all = nullptr;
  float* grad_full = nullptr;
  __nv_bfloat16* shard = nullptr;
  unsigned int* flags = nullptr;
  unsigned int* rs_flags = nullptr;  // [N+1] barrier flags of the deferred reduce-scatter (side stream)
  unsigned* ready = nullptr;   // [kMaxExperts][kMaxRanks] restore readiness (written by the pushing peers)
  float* rs_stage = nullptr;   // [E][N][S] replica grad chunks pushed by the hosts (owner side)
  // private
  void* priv = nullptr;
  float* grad_shard = nullptr;
  __nv_bfloat16* restored = nullptr;
  __nv_bfloat16 *h = nullptr, *act = nullptr, *dh = nullptr;
  __nv_bfloat16* wg = nullptr;
  float *dwg = nullptr, *dwg_partial = nullptr;
  __nv_bfloat16* dl_dense = nullptr;  // [T_max pad][kDLCols] router-gradient scatter
  int *rw_rows = nullptr, *rw_off = nullptr;
  int *topk_idx = nullptr, *intra_rank = nullptr, *blk_hist = nullptr, *blk_base = nullptr;
  float *topk_w = nullptr, *dl = nullptr;
  uint32_t* slot_dst = nullptr;
  uint8_t* layout_dev = nullptr;
  PlanTables* pt = nullptr;
  int* wave_sync = nullptr;  // grouped-GEMM wave-synchronisation counters (FSEP_WAVE_SYNC=1)
  CUtensorMap tm_w13_k128{}, tm_w2_k128{};  // K-major weight maps with 128-row boxes (CTA-pair kernel)
  CUtensorMap tm_w13_k64{};                  // ... 64-row boxes (gate-up M=128 tail tiles)
  CUtensorMap tm_x_k{}, tm_w13_k{}, tm_act_k{}, tm_w2_k{}, tm_dy_k{}, tm_w2_mn{}, tm_dh_k{}, tm_w13_mn{}, tm_dy_mn{},
      tm_act_mn{}, tm_dh_mn{}, tm_x_mn{};
  std::vector<Guard> guards;  // after every arena / private buffer
  // per-step inputs
  const __nv_bfloat16* x_in = nullptr;
};

}  // namespace
}  // namespace fsep

using namespace fsep;

extern "C" struct mp_fsep_layer {
  mp_fsep_desc d{};
  int device = 0;
  int num_sms = 148;
  int N = 1, E = 0, K = 0, H = 0, F = 0, C = 0, T_max = 0;
  long long S = 0, flat = 0;
  long long cap = 0;
  bool virt = false;
  std::vector<Rank> ranks;  // local ranks (N in virtual mode, 1 in real mode)
  PeerTable peers{};
  unsigned int** d_peer_flags = nullptr;
  __nv_bfloat16** d_tok_table = nullptr;  // [kMaxRanks] every rank's tok_rows (GEMM epilogue scatter)
  std::vector<cudaIpcMemHandle_t> opened;  // for bookkeeping
  std::vector<void*> opened_ptrs;
  bool connected = false;
  unsigned int epoch = 0;
  // layout / planner
  uint8_t* layout_host = nullptr;  // pinned E*N
  unsigned long long* R_host = nullptr;  // pinned N*E
  mp_fsep_planner* planner = nullptr;
  bool planner_pending = false;
  // streams / events
  cudaStream_t side = nullptr, plan_stream = nullptr, cap_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_restored = nullptr, ev_hist = nullptr, ev_planned = nullptr;
  static constexpr int kRing = 256;
  cudaEvent_t ev_g[kRing][4] = {};  // per-step GEMM-class timing ring (fwd begin/end, bwd begin/end)
  long long step_no = 0, stats_from = 0;
  unsigned long long slots_sum = 0;
  int T_step = 0;
  bool resident = false;       // MP_FSEP_FLAG_RESIDENT_EXPERTS: pure EP (no per-step restore / RS)
  bool restore_dirty = true;   // resident mode: hosted experts must be (re)restored
  bool local_first = false;    // MP_FSEP_FLAG_LOCAL_FIRST (non-parity routing variant)
  bool dedupe = false;         // token rows cross NVLink once per destination device (K >= 4)
  mp_fsep_layer* next = nullptr;  // chained next layer: its restore is issued after this layer's gate-up GEMM
  mp_fsep_layer* prev = nullptr;  // chained previous layer: its backward completes our deferred reduce-scatter
  // Fig.5(e) gradient-communication delay (MP_FSEP_FLAG_DEFER_RS): the owner-side half of
  // the reduce-scatter (wait for the pushes, barrier, ascending-device sum) runs on the
  // side stream under the previous layer's backward GEMMs instead of ending this backward.
  bool defer_rs = false;
  int rs_state = 0;  // 0 done, 1 pushes issued / sum pending, 2 sum enqueued on the side stream (ev_rs_done)
  unsigned int** d_peer_rs_flags = nullptr;
  unsigned int rs_epoch = 0;
  cudaEvent_t ev_rs_done = nullptr;
  bool prefetched = false;        // this layer's restore for the coming forward is already in flight
  bool restore_split = true;      // push slot 0 before dispatch, the rest after (FSEP_RESTORE_SPLIT=0: all before)
  // graph
  cudaGraphExec_t graph = nullptr;
  const void* graph_key[5] = {};
  uint64_t launches_before = 0, launches_step = 0;
  double gemm_flops_step = 0.0;
  int restore_blocks = 32;  // CTAs per (slot, peer) chunk of the restore kernel
  // Copy-engine communication (real mode, N > 1): shard restore and the grad
  // reduce-scatter gathers run as peer cudaMemcpyAsync on one stream per peer,
  // using no SMs; the forward GEMMs poll per-(slot, peer) readiness flags.
  bool ce_mode = false;
  // copy-engine lanes: ce_k streams per destination rank (1 or 2 by chunk size; FSEP_CE_STREAMS), lane d*ce_k + j;
  // slot / chunk c of destination d travels on lane d*ce_k + c % ce_k
  static constexpr int kMaxLanes = 4;
  int ce_k = 1;
  cudaStream_t ce[kMaxRanks * kMaxLanes] = {};
  cudaEvent_t ev_ce[kMaxRanks * kMaxLanes] = {};
  int lanes() const { return N * ce_k; }
  cudaEvent_t ev_wg = nullptr;
  unsigned restore_epoch = 0;
  __nv_bfloat16* peer_restored[kMaxRanks] = {};  // every rank's restored experts (push targets)
  unsigned* peer_ready[kMaxRanks] = {};
  float* peer_rs_stage[kMaxRanks] = {};
  cudaEvent_t ev_w2 = nullptr;
  uint8_t* layout_ring = nullptr;  // pinned [4][E*N] host snapshots of the layout per forward
  const uint8_t* cur_layout = nullptr;
  // optional per-phase event timing (FSEP_PHASE_TIMING=1)
  static constexpr int kPhaseRing = 64;
  bool phase_on = false;
  std::vector<std::array<cudaEvent_t, 26>> ev_p;
  std::vector<std::array<cudaEvent_t, kMaxRanks>> ev_ce_t;  // per step: last restore push to each peer landed
  double host_wait_ms = 0.0;  // host time blocked on the previous step's planner (since reset)
  // device-detected failures (fsep_types.cuh ErrWord): host-mapped words, one per cause
  unsigned* err_host = nullptr;
  unsigned* err_dev = nullptr;
  unsigned long long spin_timeout_ns = 10000000000ull;  // FSEP_SPIN_TIMEOUT_MS (barriers, readiness waits)
  // NCCL transport (FSEP_COMM=nccl, real mode): the restore as one grouped ncclSend /
  // ncclRecv exchange on the side stream (the gate-up GEMM joins it as a whole), the
  // reduce-scatter's chunks likewise into rs_stage, then the owner-side sum
  bool nccl_mode = false;
  ncclComm_t nccl = nullptr;
  cudaEvent_t ev_nccl_rs = nullptr;
  // SM push transport (FSEP_COMM=sm): the same pushes and readiness flags as the copy
  // engines, issued by push_copies_kernel on the side stream (CopyTask batches in a ring)
  bool sm_push = false;
  int push_ctas = 32;
  unsigned long long piece_bytes = 1ull << 20;
  static constexpr int kTaskRing = 16;
  int task_cap = 0, task_next = 0;
  CopyTask* task_host = nullptr;  // pinned [kTaskRing][task_cap]
  CopyTask* task_dev = nullptr;   // [kTaskRing][task_cap]
  unsigned* done_dev = nullptr;   // [kTaskRing][task_cap]
  cudaEvent_t ev_task[kTaskRing] = {};
  const unsigned char** d_guards = nullptr;  // every local rank's buffer guards (device table)
  int n_guards = 0;
  int* d_guard_bad = nullptr;
  int drop_flag = -1;  // test hook (mp_fsep_layer_debug_inject "drop_restore_flag"): source rank whose
                       // next slot-0 readiness flag is not written
};

namespace {
enum Phase : int {
  kPhFwdBegin = 0,
  kPhParamBarrier,
  kPhRouter,
  kPhRBarrier,
  kPhPlan,
  kPhDispatch,
  kPhDispatchBarrier,
  kPhRestoreWait,
  kPhFwdGateUp,  // gate-up GEMM done (the down GEMM follows)
  kPhFwdGemm,
  kPhFwdGemmBarrier,
  kPhCombine,
  kPhCombineBwd,
  kPhCombineBwdBarrier,
  kPhBwdGemm,
  kPhRsPushWait,  // own reduce-scatter pushes landed (copy-engine mode)
  kPhRsBarrier,   // everyone's pushes landed
  kPhBwdGemmBarrier,
  kPhUnpermute,
  kPhGradRS,
  kPhRestoreBegin,  // side stream
  kPhRestoreEnd,
  kPhStepBegin,  // top of the forward, before the layout snapshot / H2D
  kPhCount,
  kPhHistD2H = kPhCount,  // R copied to the host (main stream; extra ring slot)
  kPhPlanned,             // planner callback done (planner stream; extra ring slot)
};

// cuStreamWriteValue32 through the runtime's driver entry point (no libcuda link).
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValueFn write_value_fn() {
  static WriteValueFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<WriteValueFn>(nullptr);
    return reinterpret_cast<WriteValueFn>(p);
  }();
  return fn;
}

// Ascending list of experts hosted by device d under layout A (E x N).
std::vector<int> hosted_experts(const uint8_t* A, int E, int N, int d) {
  std::vector<int> out;
  for (int e = 0; e < E; ++e)
    if (A[e * N + d]) out.push_back(e);
  return out;
}

// NVTX (header-only v3: no-ops unless a tool is attached): an instantaneous marker
// at every phase boundary on the host timeline, named after the phase that ends
// there, and ranges around the public forward / backward / graph_step calls
// (NvtxRange below), so ncu --nvtx / nsys attribute each kernel to its stage.
const char* phase_name(int phase) {
  static const char* const kNames[] = {
      "fsep:fwd_begin",      "fsep:param_barrier", "fsep:router",           "fsep:R_barrier",
      "fsep:plan",           "fsep:dispatch",      "fsep:dispatch_barrier", "fsep:restore_wait",
      "fsep:fwd_gemm_gateup", "fsep:fwd_gemm_down", "fsep:fwd_barrier",     "fsep:combine",
      "fsep:combine_bwd",    "fsep:combine_bwd_barrier", "fsep:bwd_gemms",  "fsep:rs_push_wait",
      "fsep:rs_barrier",     "fsep:bwd_barrier",   "fsep:unpermute",        "fsep:grad_rs",
      "fsep:restore_begin",  "fsep:restore_end",   "fsep:step_begin",       "fsep:hist_d2h",
      "fsep:planned"};
  static_assert(sizeof(kNames) / sizeof(kNames[0]) == kPhCount + 2, "one NVTX name per phase");
  return phase >= 0 && phase < kPhCount + 2 ? kNames[phase] : "fsep:?";
}

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void mark(mp_fsep_layer& L, cudaStream_t st, int phase) {
  nvtxMarkA(phase_name(phase));
  if (!L.phase_on) return;
  cudaEventRecord(L.ev_p[static_cast<size_t>(L.step_no % mp_fsep_layer::kPhaseRing)][phase], st);
}
}  // namespace

namespace {

using Layer = mp_fsep_layer;

void build_maps(Layer& L, Rank& r) {
  const int H = L.H, F = L.F, C = L.C;
  const uint64_t cap = static_cast<uint64_t>(L.cap);
  r.tm_x_k = make_tmap_2d(r.x_rows, H, cap, H, 64, 128);
  r.tm_act_k = make_tmap_2d(r.act, F, cap, F, 64, 128);
  r.tm_dy_k = make_tmap_2d(r.dy_rows, H, cap, H, 64, 128);
  r.tm_dh_k = make_tmap_2d(r.dh, 2 * F, cap, 2 * F, 64, 128);
  r.tm_dy_mn = make_tmap_2d(r.dy_rows, H, cap, H, 64, 64);
  r.tm_act_mn = make_tmap_2d(r.act, F, cap, F, 64, 64);
  r.tm_dh_mn = make_tmap_2d(r.dh, 2 * F, cap, 2 * F, 64, 64);
  r.tm_x_mn = make_tmap_2d(r.x_rows, H, cap, H, 64, 64);
  const __nv_bfloat16* w13 = r.restored;
  const __nv_bfloat16* w2 = r.restored + 2LL * F * H;
  r.tm_w13_k = make_tmap_3d(w13, H, 2 * F, C, H, L.flat, 64, 256);
  r.tm_w2_k = make_tmap_3d(w2, F, H, C, F, L.flat, 64, 256);
  r.tm_w13_k128 = make_tmap_3d(w13, H, 2 * F, C, H, L.flat, 64, 128);
  r.tm_w13_k64 = make_tmap_3d(w13, H, 2 * F, C, H, L.flat, 64, 64);
  r.tm_w2_k128 = make_tmap_3d(w2, F, H, C, F, L.flat, 64, 128);
  r.tm_w2_mn = make_tmap_3d(w2, F, H, C, F, L.flat, 64, 64);
  r.tm_w13_mn = make_tmap_3d(w13, H, 2 * F, C, H, L.flat, 64, 64);
}

void allocate_rank(Layer& L, Rank& r) {
  const size_t H = L.H, F = L.F, E = L.E, C = L.C, N = L.N, T = L.T_max, K = L.K;
  const size_t cap = static_cast<size_t>(L.cap);
  const size_t S = static_cast<size_t>(L.S), flat = static_cast<size_t>(L.flat);
  const size_t nblk = (T + kBlockTokens - 1) / kBlockTokens;
  const bool push = L.ce_mode;
  const bool multi = N > 1;
  const int splits = router_wgrad_splits(static_cast<int>(T));
  // Each carve runs twice: on a null base to measure the bytes (guards and 256-B
  // alignment included), then on the allocation.  Identical on every rank, so peer
  // offsets match.
  auto carve_arena = [&](Carver& ca) {  // peer-visible
    r.x_rows = ca.take<__nv_bfloat16>(cap * H, "x_rows");
    r.dy_rows = ca.take<__nv_bfloat16>(cap * H, "dy_rows");
    r.tok_rows = ca.take<__nv_bfloat16>(T * K * H, "tok_rows");
    r.row_src = ca.take<int>(cap, "row_src");
    if (L.dedupe) {
      r.stage = ca.take<__nv_bfloat16>(N * T * H, "stage");
      r.row_w = ca.take<float>(cap, "row_w");
    }
    r.R_all = ca.take<unsigned long long>(N * E, "R_all");
    r.grad_full = ca.take<float>(C * flat, "grad_full");
    r.shard = ca.take<__nv_bfloat16>(E * S, "shard");
    r.flags = ca.take<unsigned int>(N + 1, "flags");
    r.rs_flags = ca.take<unsigned int>(N + 1, "rs_flags");
    if (push) {
      r.restored = ca.take<__nv_bfloat16>(C * flat, "restored");  // push target
      r.ready = ca.take<unsigned>(kMaxExperts * kMaxRanks, "ready");
    }
    if (push || L.nccl_mode) r.rs_stage = ca.take<float>(E * N * S, "rs_stage");
  };
  auto carve_private = [&](Carver& cp) {
    if (multi) {
      r.grad_shard = cp.take<float>(E * S, "grad_shard");
      if (!push) r.restored = cp.take<__nv_bfloat16>(C * flat, "restored");
    }
    r.h = cp.take<__nv_bfloat16>(cap * 2 * F, "h");
    r.act = cp.take<__nv_bfloat16>(cap * F, "act");
    r.dh = cp.take<__nv_bfloat16>(cap * 2 * F, "dh");
    r.wg = cp.take<__nv_bfloat16>(E * H, "wg");
    r.dwg = cp.take<float>(E * H, "dwg");
    r.dwg_partial = cp.take<float>(static_cast<size_t>(splits) * kDLCols * H, "dwg_partial");  // split-K partials
    r.dl_dense = cp.take<__nv_bfloat16>((T + 127) / 128 * 128 * kDLCols, "dl_dense");
    r.rw_rows = cp.take<int>(splits, "rw_rows");
    r.rw_off = cp.take<int>(splits, "rw_off");
    r.topk_idx = cp.take<int>(T * K, "topk_idx");
    r.intra_rank = cp.take<int>(T * K, "intra_rank");
    r.topk_w = cp.take<float>(T * K, "topk_w");
    r.dl = cp.take<float>(T * K, "dl");
    r.slot_dst = cp.take<uint32_t>(T * K, "slot_dst");
    r.blk_hist = cp.take<int>(nblk * E, "blk_hist");
    r.blk_base = cp.take<int>(nblk * E, "blk_base");
    r.layout_dev = cp.take<uint8_t>(E * N, "layout_dev");
    r.pt = cp.take<PlanTables>(1, "pt");
    r.wave_sync = cp.take<int>(kWaveSyncMax, "wave_sync");
  };
  std::vector<Guard> scratch;
  Carver measure_a{nullptr, &scratch}, measure_p{nullptr, &scratch};
  carve_arena(measure_a);
  carve_private(measure_p);
  r.arena_bytes = align_up(measure_a.off, 2 << 20);
  const size_t priv_bytes = align_up(measure_p.off, 2 << 20);
  CK(cudaMalloc(&r.arena, r.arena_bytes));
  CK(cudaMemset(r.arena, 0, r.arena_bytes));
  CK(cudaMalloc(&r.priv, priv_bytes));
  CK(cudaMemset(r.priv, 0, priv_bytes));
  r.guards.clear();
  Carver ca{static_cast<char*>(r.arena), &r.guards};
  carve_arena(ca);
  Carver cp{static_cast<char*>(r.priv), &r.guards};
  carve_private(cp);
  if (!multi) {
    r.grad_shard = r.grad_full;  // one device: the shard IS the full expert set (C == E)
    r.restored = r.shard;
  }
  // fill the guards (the arenas were zeroed above)
  for (const Guard& g : r.guards) CK(cudaMemset(const_cast<unsigned char*>(g.at), kGuardByte, kGuardBytes));
  build_maps(L, r);
}

void finish_peers(Layer& L) {
  // virtual mode: all ranks local; real mode: filled by connect()
  if (L.virt) {
    for (int p = 0; p < L.N; ++p) {
      Rank& r = L.ranks[p];
      L.peers.x_rows[p] = r.x_rows;
      L.peers.dy_rows[p] = r.dy_rows;
      L.peers.tok_rows[p] = r.tok_rows;
      L.peers.row_src[p] = r.row_src;
      L.peers.stage[p] = r.stage;
      L.peers.row_w[p] = r.row_w;
      L.peers.R_all[p] = r.R_all;
      L.peers.grad_full[p] = r.grad_full;
      L.peers.shard[p] = r.shard;
      if (L.ce_mode) {  // virtual copy-engine mode: push targets are the emulated ranks' arenas
        L.peer_restored[p] = r.restored;
        L.peer_ready[p] = r.ready;
        L.peer_rs_stage[p] = r.rs_stage;
      }
    }
  }
  L.peers.row_capacity = static_cast<uint64_t>(L.cap);
}

void barrier(Layer& L, cudaStream_t st) {
  if (L.virt || L.N == 1) return;  // stream order is the barrier on one GPU
  launch_peer_barrier(L.d_peer_flags, L.N, L.ranks[0].rank, ++L.epoch, L.err_dev, L.spin_timeout_ns, st);
}

// Owner-side completion of a reduce-scatter whose pushes were issued by L's backward:
// on L's side stream wait for L's own pushes, then (real mode) a barrier on the
// separate rs flags (everyone's pushes landed), then the ascending-device sum.
void finish_rs_async(Layer& L) {
  if (L.rs_state != 1) return;
  for (int o = 0; o < L.lanes(); ++o) CK(cudaStreamWaitEvent(L.side, L.ev_ce[o], 0));
  if (!L.virt && L.N > 1)
    launch_peer_barrier(L.d_peer_rs_flags, L.N, L.ranks[0].rank, ++L.rs_epoch, L.err_dev, L.spin_timeout_ns, L.side);
  for (Rank& r : L.ranks)
    launch_grad_rs_sum(r.pt, r.grad_full, r.rs_stage, L.E, L.N, r.rank, L.S, L.flat, r.grad_shard, L.side);
  CK(cudaEventRecord(L.ev_rs_done, L.side));
  L.rs_state = 2;
}

// Make L's reduced gradient shards final on `st` (finishing a still-pending deferral).
void join_rs(Layer& L, cudaStream_t st) {
  finish_rs_async(L);
  if (L.rs_state == 2) {
    CK(cudaStreamWaitEvent(st, L.ev_rs_done, 0));
    L.rs_state = 0;
  }
}

// CTA-pair (cta_group::2) kernel by default; FSEP_GEMM=single forces the 128x256 single-CTA kernel.
bool use_pair_gemm() {
  static const bool single = [] {
    const char* v = std::getenv("FSEP_GEMM");
    return v && std::string(v) == "single";
  }();
  return !single;
}

void gemm(Layer& L, GemmKind kind, const CUtensorMap& a, const CUtensorMap& b_single, const CUtensorMap& b_pair,
          const GroupedGemmArgs& g, cudaStream_t st) {
  if (use_pair_gemm() && pair_gemm_supported(kind, g))
    launch_grouped_gemm_pair(kind, a, b_pair, g, L.num_sms, st);
  else
    launch_grouped_gemm(kind, a, b_single, g, L.num_sms, st);
}

GroupedGemmArgs gemm_args(Layer& L, Rank& r) {
  GroupedGemmArgs g{};
  g.num_groups = L.C;
  g.group_rows = r.pt->seg_rows_pad;
  g.group_off = r.pt->seg_off;
  g.wave_sync = r.wave_sync;
  g.err = L.err_dev;
  g.ready_timeout_ns = L.spin_timeout_ns;
  return g;
}

// Copy-engine mode: snapshot this step's layout on the host (waiting for the
// previous step's planner callback) and ship it to the device on `st`.
void snapshot_layout(Layer& L, cudaStream_t st) {
  const int E = L.E, N = L.N;
  if (L.planner_pending) {
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaEventSynchronize(L.ev_planned));
    L.host_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  uint8_t* snap = L.layout_ring + (L.step_no % 4) * static_cast<size_t>(E) * N;
  std::memcpy(snap, L.layout_host, static_cast<size_t>(E) * N);
  L.cur_layout = snap;
  for (Rank& r : L.ranks) CK(cudaMemcpyAsync(r.layout_dev, snap, static_cast<size_t>(E) * N, cudaMemcpyHostToDevice, st));
}

// SM push transport: copy `tasks` with push_copies_kernel on the side stream after
// `st`'s work so far, and record every ev_ce[d] after it (same joins as the copy engines).
void sm_push(Layer& L, cudaStream_t st, std::vector<CopyTask>& tasks) {
  if (tasks.empty()) return;
  if (static_cast<int>(tasks.size()) > L.task_cap) throw Error(ErrorKind::device, "sm push: task batch too large");
  unsigned pieces = 0;
  for (CopyTask& t : tasks) {
    t.first_piece = pieces;
    pieces += static_cast<unsigned>((t.bytes + L.piece_bytes - 1) / L.piece_bytes);
  }
  const int k = L.task_next++ % Layer::kTaskRing;
  CK(cudaEventSynchronize(L.ev_task[k]));  // the ring slot's previous upload is done
  CopyTask* h = L.task_host + static_cast<size_t>(k) * L.task_cap;
  CopyTask* d = L.task_dev + static_cast<size_t>(k) * L.task_cap;
  std::memcpy(h, tasks.data(), tasks.size() * sizeof(CopyTask));
  CK(cudaEventRecord(L.ev_fork, st));
  CK(cudaStreamWaitEvent(L.side, L.ev_fork, 0));
  CK(cudaMemcpyAsync(d, h, tasks.size() * sizeof(CopyTask), cudaMemcpyHostToDevice, L.side));
  CK(cudaEventRecord(L.ev_task[k], L.side));
  launch_push_copies(d, static_cast<int>(tasks.size()), pieces, L.piece_bytes,
                     L.done_dev + static_cast<size_t>(k) * L.task_cap, L.push_ctas, L.side);
  for (int p = 0; p < L.lanes(); ++p) CK(cudaEventRecord(L.ev_ce[p], L.side));
}

// Push restore: each local rank's chunk of every expert goes straight into the
// restored slot of each rank that hosts it (own slots first), and a flag written
// into the destination's memory after each copy releases that (slot, source)
// pair to the destination's gate-up GEMM producer.  Ordered after `st`'s work.
// Slots [c0, c1) of every destination; c0 == 0 opens a new restore epoch.
// Real mode: one local rank, one copy-engine stream per destination GPU.
// Virtual mode (MP_FSEP_FLAG_COPY_ENGINE): the same copies and flags between the
// emulated ranks' arenas on one GPU, stream ce[d] carrying every push into d.
void push_restore(Layer& L, cudaStream_t st, int c0 = 0, int c1 = kMaxExperts) {
  const int E = L.E, N = L.N;
  if (c0 == 0) {
    ++L.restore_epoch;
    mark(L, st, kPhRestoreBegin);
  }
  if (L.sm_push) {  // slot-major task order: slot c of every destination before slot c+1
    std::vector<std::vector<int>> theirs(N);
    for (int d = 0; d < N; ++d) theirs[d] = hosted_experts(L.cur_layout, E, N, d);
    std::vector<CopyTask> tasks;
    for (int c = c0; c < std::min(c1, L.C); ++c)
      for (Rank& r : L.ranks)
        for (int q = 0; q < N; ++q) {
          const int d = (r.rank + q) % N;
          if (c >= static_cast<int>(theirs[d].size())) continue;
          CopyTask t{};
          t.src = r.shard + static_cast<long long>(theirs[d][c]) * L.S;
          t.dst = L.peer_restored[d] + static_cast<long long>(c) * L.flat + static_cast<long long>(r.rank) * L.S;
          t.bytes = static_cast<unsigned long long>(L.S) * 2;
          t.flag = L.peer_ready[d] + c * N + r.rank;
          t.flag_val = L.restore_epoch;
          if (c == 0 && L.drop_flag == r.rank && d != r.rank) {  // test hook: this flag never arrives
            L.drop_flag = -1;
            t.flag = nullptr;
          }
          tasks.push_back(t);
        }
    sm_push(L, st, tasks);
    if (L.phase_on)
      for (int d = 0; d < N; ++d)
        cudaEventRecord(L.ev_ce_t[static_cast<size_t>(L.step_no % mp_fsep_layer::kPhaseRing)][d], L.side);
    return;
  }
  CK(cudaEventRecord(L.ev_fork, st));
  for (int d = 0; d < L.lanes(); ++d) CK(cudaStreamWaitEvent(L.ce[d], L.ev_fork, 0));
  for (Rank& r : L.ranks) {
    for (int q = 0; q < N; ++q) {
      const int d = (r.rank + q) % N;
      const std::vector<int> theirs = hosted_experts(L.cur_layout, E, N, d);
      for (int c = c0; c < std::min(c1, static_cast<int>(theirs.size())); ++c) {
        CK(cudaMemcpyAsync(L.peer_restored[d] + static_cast<long long>(c) * L.flat + static_cast<long long>(r.rank) * L.S,
                           r.shard + static_cast<long long>(theirs[c]) * L.S, static_cast<size_t>(L.S) * 2,
                           cudaMemcpyDeviceToDevice, L.ce[d * L.ce_k + c % L.ce_k]));
        if (c == 0 && L.drop_flag == r.rank && d != r.rank) {  // test hook: this flag never arrives
          L.drop_flag = -1;
          continue;
        }
        if (write_value_fn()(L.ce[d * L.ce_k + c % L.ce_k], reinterpret_cast<CUdeviceptr>(L.peer_ready[d] + c * N + r.rank),
                             L.restore_epoch, 0) != CUDA_SUCCESS)
          throw Error(ErrorKind::device, "cuStreamWriteValue32 failed");
      }
    }
  }
  for (int d = 0; d < N; ++d) {
    for (int j = 0; j < L.ce_k; ++j) CK(cudaEventRecord(L.ev_ce[d * L.ce_k + j], L.ce[d * L.ce_k + j]));
    if (L.phase_on) cudaEventRecord(L.ev_ce_t[static_cast<size_t>(L.step_no % mp_fsep_layer::kPhaseRing)][d], L.ce[d * L.ce_k]);
  }
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(ErrorKind::device, std::string(what) + ": " + ncclGetErrorString(r));
}

// NCCL transport: this rank's chunk of every expert hosted by d goes to d with ncclSend,
// chunk p of every expert hosted here arrives from p with ncclRecv straight into its
// restored slot (one group on the side stream, after `st`'s work; ev_restored after it).
void nccl_restore(Layer& L, cudaStream_t st) {
  const int E = L.E, N = L.N;
  Rank& r = L.ranks[0];
  CK(cudaEventRecord(L.ev_fork, st));
  CK(cudaStreamWaitEvent(L.side, L.ev_fork, 0));
  mark(L, L.side, kPhRestoreBegin);
  const std::vector<int> mine = hosted_experts(L.cur_layout, E, N, r.rank);
  for (int c = 0; c < static_cast<int>(mine.size()); ++c)  // own chunk: local copy
    CK(cudaMemcpyAsync(r.restored + static_cast<long long>(c) * L.flat + static_cast<long long>(r.rank) * L.S,
                       r.shard + static_cast<long long>(mine[c]) * L.S, static_cast<size_t>(L.S) * 2,
                       cudaMemcpyDeviceToDevice, L.side));
  nccl_check(ncclGroupStart(), "ncclGroupStart");
  for (int q = 1; q < N; ++q) {
    const int d = (r.rank + q) % N, p = (r.rank + N - q) % N;
    for (int e : hosted_experts(L.cur_layout, E, N, d))
      nccl_check(ncclSend(r.shard + static_cast<long long>(e) * L.S, static_cast<size_t>(L.S), ncclBfloat16, d, L.nccl,
                          L.side), "ncclSend");
    for (int c = 0; c < static_cast<int>(mine.size()); ++c)
      nccl_check(ncclRecv(r.restored + static_cast<long long>(c) * L.flat + static_cast<long long>(p) * L.S,
                          static_cast<size_t>(L.S), ncclBfloat16, p, L.nccl, L.side), "ncclRecv");
  }
  nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  mark(L, L.side, kPhRestoreEnd);
  CK(cudaEventRecord(L.ev_restored, L.side));
}

// NCCL reduce-scatter exchange: this rank's replica chunk o of every hosted expert to its
// owner o; chunk `rank` of every expert from each of its other hosts into rs_stage.
void nccl_grad_exchange(Layer& L, cudaStream_t st) {
  const int E = L.E, N = L.N;
  Rank& r = L.ranks[0];
  CK(cudaEventRecord(L.ev_fork, st));
  CK(cudaStreamWaitEvent(L.side, L.ev_fork, 0));
  const std::vector<int> mine = hosted_experts(L.cur_layout, E, N, r.rank);
  nccl_check(ncclGroupStart(), "ncclGroupStart");
  for (int q = 1; q < N; ++q) {
    const int o = (r.rank + q) % N, p = (r.rank + N - q) % N;
    for (int c = 0; c < static_cast<int>(mine.size()); ++c)
      nccl_check(ncclSend(r.grad_full + static_cast<long long>(c) * L.flat + static_cast<long long>(o) * L.S,
                          static_cast<size_t>(L.S), ncclFloat32, o, L.nccl, L.side), "ncclSend");
    for (int e : hosted_experts(L.cur_layout, E, N, p))
      nccl_check(ncclRecv(r.rs_stage + (static_cast<long long>(e) * N + p) * L.S, static_cast<size_t>(L.S),
                          ncclFloat32, p, L.nccl, L.side), "ncclRecv");
  }
  nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  CK(cudaEventRecord(L.ev_nccl_rs, L.side));
}

void run_forward(Layer& L, const __nv_bfloat16* x, const float* bias, int T, __nv_bfloat16* y, cudaStream_t st) {
  if (T < 0 || T > L.T_max) throw Error(ErrorKind::invalid_argument, "forward: n_tokens exceeds max_tokens");
  const int E = L.E, K = L.K, H = L.H, F = L.F, N = L.N, C = L.C;
  L.T_step = T;
  mark(L, st, kPhStepBegin);
  const long long TH = static_cast<long long>(T) * H;
  // 1. layout for this step (planner result of the previous step, or set_layout)
  const bool ce = L.ce_mode;
  const bool prefetched = L.prefetched;  // chained: layout + restore already issued by the previous layer
  L.prefetched = false;
  if (ce || L.nccl_mode) {
    // Copy-engine restore needs the layout on the host: wait for the previous
    // step's planner callback (it ran right after that step's router, so the
    // host stays up to one step ahead) and snapshot it for this step.
    if (!prefetched) snapshot_layout(L, st);
  } else {
    if (L.planner_pending) CK(cudaStreamWaitEvent(st, L.ev_planned, 0));
    for (Rank& r : L.ranks)
      CK(cudaMemcpyAsync(r.layout_dev, L.layout_host, static_cast<size_t>(E) * N, cudaMemcpyHostToDevice, st));
  }
  // 2. shard restore on the side stream(s) (overlaps router + dispatch, and in
  //    copy-engine mode the forward GEMMs too: they wait per slot, not per step)
  const bool restore = N > 1 && (!L.resident || L.restore_dirty);
  if (L.resident) L.restore_dirty = false;
  mark(L, st, kPhFwdBegin);
  // peers' shards must be final (parameter load / optimizer update) before anyone gathers them
  barrier(L, st);
  mark(L, st, kPhParamBarrier);
  if (restore && ce) {
    // only slot 0 now; the other slots after dispatch, so the restore does not
    // compete with the dispatch for NVLink (slot 0 is what the GEMMs need first)
    if (!prefetched) push_restore(L, st, 0, L.restore_split ? 1 : kMaxExperts);
  } else if (restore && L.nccl_mode) {
    nccl_restore(L, st);
  } else if (restore) {
    CK(cudaEventRecord(L.ev_fork, st));
    CK(cudaStreamWaitEvent(L.side, L.ev_fork, 0));
    mark(L, L.side, kPhRestoreBegin);
    for (Rank& r : L.ranks)
      launch_restore(r.layout_dev, E, N, r.rank, C, L.S, L.flat, L.peers, r.restored, L.restore_blocks, L.side);
    mark(L, L.side, kPhRestoreEnd);
    CK(cudaEventRecord(L.ev_restored, L.side));
  }
  // 3. router + top-k + histogram, global ranks, R exchange
  const int nblk = (T + kBlockTokens - 1) / kBlockTokens;
  for (size_t v = 0; v < L.ranks.size(); ++v) {
    Rank& r = L.ranks[v];
    r.x_in = x + (L.virt ? static_cast<long long>(v) * TH : 0);
    const float* b = bias ? bias + (L.virt ? static_cast<long long>(v) * T * E : 0) : nullptr;
    launch_router(RouterArgs{r.x_in, r.wg, b, T, H, E, K, r.topk_idx, r.topk_w, r.intra_rank, r.blk_hist}, st);
    launch_block_scan(r.blk_hist, nblk, E, r.blk_base, L.peers, r.rank, N, st);
  }
  mark(L, st, kPhRouter);
  barrier(L, st);
  mark(L, st, kPhRBarrier);
  // 4. device lite routing + receive layout; dispatch
  for (Rank& r : L.ranks) {
    launch_plan(r.R_all, r.layout_dev, E, N, r.rank, r.pt, L.cap, L.local_first, L.err_dev, st);
    launch_zero_pad(r.pt, C, H, r.x_rows, r.dy_rows, r.row_src, st);
  }
  mark(L, st, kPhPlan);
  // histogram -> host planner (async, off the critical path)
  CK(cudaMemcpyAsync(L.R_host, L.ranks[0].R_all, static_cast<size_t>(N) * E * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(L.ev_hist, st));
  mark(L, st, kPhHistD2H);
  if (L.planner) {
    CK(cudaStreamWaitEvent(L.plan_stream, L.ev_hist, 0));
    CK(cudaLaunchHostFunc(
        L.plan_stream,
        [](void* p) {
          Layer* l = static_cast<Layer*>(p);
          // errors cannot propagate from a host node; keep the previous layout on failure
          if (mp_fsep_planner_observe(l->planner, reinterpret_cast<const uint64_t*>(l->R_host)) == MP_OK) mp_fsep_planner_next(l->planner, l->layout_host);
        },
        &L));
    CK(cudaEventRecord(L.ev_planned, L.plan_stream));
    mark(L, L.plan_stream, kPhPlanned);
    L.planner_pending = true;
  }
  for (Rank& r : L.ranks)
    launch_dispatch(DispatchArgs{r.x_in, T, H, K, E, r.topk_idx, r.intra_rank, r.blk_base, r.pt, L.peers, r.slot_dst,
                                 r.rank, r.topk_w, L.T_max, L.dedupe},
                    st);
  mark(L, st, kPhDispatch);
  if (restore && ce && !prefetched && L.restore_split) push_restore(L, st, 1, kMaxExperts);
  barrier(L, st);
  if (L.dedupe)  // token rows that crossed NVLink once per device -> this rank's slot rows
    for (Rank& r : L.ranks)
      launch_expand_rows(r.pt, L.cap, r.row_src, r.stage, nullptr, r.rank, H, K, L.T_max, r.x_rows, L.num_sms, st);
  mark(L, st, kPhDispatchBarrier);
  // 5. expert FFN on the restored experts
  if (restore && !ce) CK(cudaStreamWaitEvent(st, L.ev_restored, 0));
  mark(L, st, kPhRestoreWait);
  CK(cudaEventRecord(L.ev_g[L.step_no % Layer::kRing][0], st));
  for (Rank& r : L.ranks) {
    GroupedGemmArgs g = gemm_args(L, r);
    if (restore && ce) {  // per-(slot, peer) readiness instead of a whole-restore join
      g.ready = r.ready;
      g.ready_epoch = L.restore_epoch;
      g.ready_n = N;
    }
    g.N = 2 * F;
    g.K = H;
    g.out = r.h;
    g.ldo = 2 * F;
    g.out2 = r.act;
    g.ldo2 = F;
    g.b64 = &r.tm_w13_k64;
    gemm(L, GemmKind::kFwdGateUp, r.tm_x_k, r.tm_w13_k, r.tm_w13_k128, g, st);
    if (&r == &L.ranks.back()) {
      mark(L, st, kPhFwdGateUp);
      // Fig.5 schedule: the next layer's expert restore travels on the copy engines
      // while this layer's down GEMM, combine and the next layer's router/dispatch
      // run.  Issued after the gate-up GEMM, which has waited for all of this
      // layer's restored slots, so the two restores never share the copy engines
      // (safe: every rank has passed this step's parameter barrier, so all of the
      // previous step's work is complete).
      if (L.next && L.next->ce_mode && !L.next->prefetched && (!L.next->resident || L.next->restore_dirty)) {
        Layer& nx = *L.next;
        snapshot_layout(nx, st);
        push_restore(nx, st);
        nx.prefetched = true;
      }
    }
    GroupedGemmArgs g2 = g;
    g2.N = H;
    g2.K = F;
    g2.out = nullptr;  // rows go straight to the token owners' tok_rows (epilogue scatter)
    g2.ldo = H;
    g2.row_src = r.row_src;
    g2.scatter = L.d_tok_table;
    g2.scatter_rows = static_cast<long long>(L.T_max) * K;
    g2.out2 = nullptr;
    g2.ldo2 = 0;
    gemm(L, GemmKind::kFwdDown, r.tm_act_k, r.tm_w2_k, r.tm_w2_k128, g2, st);
  }
  if (restore && ce) {
    for (int p = 0; p < L.lanes(); ++p) CK(cudaStreamWaitEvent(st, L.ev_ce[p], 0));  // join (long complete)
    mark(L, st, kPhRestoreEnd);
  }
  CK(cudaEventRecord(L.ev_g[L.step_no % Layer::kRing][1], st));
  mark(L, st, kPhFwdGemm);
  barrier(L, st);
  mark(L, st, kPhFwdGemmBarrier);
  // 6. combine
  for (size_t v = 0; v < L.ranks.size(); ++v) {
    Rank& r = L.ranks[v];
    launch_combine(T, H, K, r.topk_w, r.tok_rows, y + (L.virt ? static_cast<long long>(v) * TH : 0), st);
  }
  mark(L, st, kPhCombine);
}

void run_backward(Layer& L, const __nv_bfloat16* dy, __nv_bfloat16* dx, cudaStream_t st) {
  const int E = L.E, K = L.K, H = L.H, F = L.F, N = L.N, T = L.T_step;
  const long long TH = static_cast<long long>(T) * H;
  // This layer's own reduce-scatter of the previous step still pending (its predecessor's
  // backward never ran): complete it before this backward overwrites grad_full.
  if (L.rs_state != 0) {
    CK(cudaEventRecord(L.ev_fork, st));
    CK(cudaStreamWaitEvent(L.side, L.ev_fork, 0));
    join_rs(L, st);
  }
  // Fig.5(e): the next layer (already back-propagated this step) deferred the owner-side
  // half of its reduce-scatter; it runs on that layer's side stream under this layer's GEMMs.
  Layer* deferred = (L.next && L.next->rs_state == 1) ? L.next : nullptr;
  if (deferred) {
    CK(cudaEventRecord(L.ev_fork, st));
    CK(cudaStreamWaitEvent(deferred->side, L.ev_fork, 0));
    finish_rs_async(*deferred);
  }
  for (size_t v = 0; v < L.ranks.size(); ++v) {
    Rank& r = L.ranks[v];
    launch_combine_bwd(T, H, K, E, dy + (L.virt ? static_cast<long long>(v) * TH : 0), r.topk_w, r.topk_idx, r.tok_rows,
                       r.slot_dst, L.peers, r.dl, r.dl_dense, r.rw_rows, r.rw_off, r.rank, L.T_max, L.dedupe, st);
    launch_router_wgrad(r.x_in, T, H, E, r.dl_dense, L.T_max, r.rw_rows, r.rw_off, r.dwg_partial, r.dwg, L.num_sms,
                        st);
  }
  mark(L, st, kPhCombineBwd);
  barrier(L, st);
  if (L.dedupe)  // dout rows that crossed NVLink once per device -> w_k-scaled dY slot rows
    for (Rank& r : L.ranks)
      launch_expand_rows(r.pt, L.cap, r.row_src, r.stage, r.row_w, r.rank, H, K, L.T_max, r.dy_rows, L.num_sms, st);
  mark(L, st, kPhCombineBwdBarrier);
  CK(cudaEventRecord(L.ev_g[L.step_no % Layer::kRing][2], st));
  // Weight gradients first: in copy-engine mode their reduce-scatter pushes run
  // on the copy engines underneath the GEMMs that follow.
  const bool rs = N > 1 && !L.resident;  // pure EP: gradients stay whole on their single host
  const bool ce_rs = L.ce_mode && rs;
  // the previous chained layer's backward (run next) completes the reduce-scatter
  const bool defer = ce_rs && L.defer_rs && L.prev != nullptr;
  // Push this rank's replica-gradient chunks [lo, hi) of the flat vector to their
  // owners' staging rows (copy engines, one stream per owner), after `ev`.
  auto push_grads = [&](cudaEvent_t ev, long long lo, long long hi) {
    if (L.sm_push) {
      std::vector<CopyTask> tasks;
      for (Rank& r : L.ranks) {
        const std::vector<int> mine = hosted_experts(L.cur_layout, E, N, r.rank);
        for (int q = 1; q < N; ++q) {
          const int o = (r.rank + q) % N;
          const long long a = std::max(lo, static_cast<long long>(o) * L.S);
          const long long b = std::min(hi, static_cast<long long>(o + 1) * L.S);
          if (a >= b) continue;
          for (int c = 0; c < static_cast<int>(mine.size()); ++c) {
            CopyTask t{};
            t.src = r.grad_full + static_cast<long long>(c) * L.flat + a;
            t.dst = L.peer_rs_stage[o] + (static_cast<long long>(mine[c]) * N + r.rank) * L.S + (a - o * L.S);
            t.bytes = static_cast<unsigned long long>(b - a) * 4;
            tasks.push_back(t);
          }
        }
      }
      (void)ev;  // sm_push orders after st's work (the wgrad GEMM) itself
      sm_push(L, st, tasks);
      return;
    }
    for (int o = 0; o < L.lanes(); ++o) CK(cudaStreamWaitEvent(L.ce[o], ev, 0));
    for (Rank& r : L.ranks) {
      const std::vector<int> mine = hosted_experts(L.cur_layout, E, N, r.rank);
      for (int q = 1; q < N; ++q) {
        const int o = (r.rank + q) % N;
        const long long a = std::max(lo, static_cast<long long>(o) * L.S);
        const long long b = std::min(hi, static_cast<long long>(o + 1) * L.S);
        if (a >= b) continue;
        for (int c = 0; c < static_cast<int>(mine.size()); ++c)
          CK(cudaMemcpyAsync(L.peer_rs_stage[o] + (static_cast<long long>(mine[c]) * N + r.rank) * L.S + (a - o * L.S),
                             r.grad_full + static_cast<long long>(c) * L.flat + a, static_cast<size_t>(b - a) * 4,
                             cudaMemcpyDeviceToDevice, L.ce[o * L.ce_k + c % L.ce_k]));
      }
    }
    for (int o = 0; o < L.lanes(); ++o) CK(cudaEventRecord(L.ev_ce[o], L.ce[o]));
  };
  const long long w2_lo = 2LL * F * H;
  // Order: dH (SwiGLU' fused), dW13, dW2, dX.  The W13 part of the replica
  // gradient chunks (2/3 of the reduce-scatter bytes) is pushed as soon as dW13 is
  // done and travels under dW2 + dX; the W2 part travels under dX.
  for (Rank& r : L.ranks) {
    GroupedGemmArgs g = gemm_args(L, r);  // dAct -> dH (SwiGLU backward fused)
    g.N = F;
    g.K = H;
    g.out = r.dh;
    g.ldo = 2 * F;
    g.aux = r.h;
    g.ld_aux = 2 * F;
    gemm(L, GemmKind::kBwdDownDgrad, r.tm_dy_k, r.tm_w2_mn, r.tm_w2_mn, g, st);
    GroupedGemmArgs g4 = gemm_args(L, r);  // dW13 = dH^T X
    g4.M = 2 * F;
    g4.N = H;
    g4.out = r.grad_full;
    g4.ldo = H;
    g4.out_group_stride = L.flat;
    gemm(L, GemmKind::kBwdWgrad, r.tm_dh_mn, r.tm_x_mn, r.tm_x_mn, g4, st);
  }
  if (ce_rs) {
    CK(cudaEventRecord(L.ev_wg, st));
    push_grads(L.ev_wg, 0, w2_lo);
  }
  for (Rank& r : L.ranks) {
    GroupedGemmArgs g3 = gemm_args(L, r);  // dW2 = dY^T act
    g3.M = H;
    g3.N = F;
    g3.out = r.grad_full + 2LL * F * H;
    g3.ldo = F;
    g3.out_group_stride = L.flat;
    gemm(L, GemmKind::kBwdWgrad, r.tm_dy_mn, r.tm_act_mn, r.tm_act_mn, g3, st);
  }
  if (ce_rs) {
    CK(cudaEventRecord(L.ev_w2, st));
    push_grads(L.ev_w2, w2_lo, L.flat);
  }
  const bool nccl_rs = rs && L.nccl_mode;
  if (nccl_rs) nccl_grad_exchange(L, st);  // under the dX GEMM (NCCL's CTAs get SMs as the GEMM frees them)
  for (Rank& r : L.ranks) {
    GroupedGemmArgs g2 = gemm_args(L, r);  // dX rows
    g2.N = H;
    g2.K = 2 * F;
    g2.out = nullptr;  // dX rows go straight to the token owners' tok_rows (y is dead by now)
    g2.ldo = H;
    g2.row_src = r.row_src;
    g2.scatter = L.d_tok_table;
    g2.scatter_rows = static_cast<long long>(L.T_max) * K;
    gemm(L, GemmKind::kBwdUpDgrad, r.tm_dh_k, r.tm_w13_mn, r.tm_w13_mn, g2, st);
  }
  CK(cudaEventRecord(L.ev_g[L.step_no % Layer::kRing][3], st));
  mark(L, st, kPhBwdGemm);
  if (defer) {
    mark(L, st, kPhRsPushWait);
    barrier(L, st);  // every rank's dX GEMM stored its dX rows into our tok_rows
    mark(L, st, kPhRsBarrier);
    L.rs_state = 1;
  } else if (ce_rs) {
    for (int o = 0; o < L.lanes(); ++o) CK(cudaStreamWaitEvent(st, L.ev_ce[o], 0));  // own pushes landed
    mark(L, st, kPhRsPushWait);
    // ... and everyone else's: this barrier also orders every rank's dX GEMM (whose
    // epilogue stored dX rows into our tok_rows) before the unpermute below
    barrier(L, st);
    mark(L, st, kPhRsBarrier);
    for (Rank& r : L.ranks)
      launch_grad_rs_sum(r.pt, r.grad_full, r.rs_stage, E, N, r.rank, L.S, L.flat, r.grad_shard, st);
  } else {
    mark(L, st, kPhRsPushWait);
    barrier(L, st);
    mark(L, st, kPhRsBarrier);
  }
  mark(L, st, kPhBwdGemmBarrier);
  for (size_t v = 0; v < L.ranks.size(); ++v) {
    Rank& r = L.ranks[v];
    launch_unpermute_bwd(T, H, K, r.topk_idx, r.dl, r.tok_rows, r.wg, dx + (L.virt ? static_cast<long long>(v) * TH : 0),
                         st);
  }
  mark(L, st, kPhUnpermute);
  if (nccl_rs) {
    CK(cudaStreamWaitEvent(st, L.ev_nccl_rs, 0));
    for (Rank& r : L.ranks)
      launch_grad_rs_sum(r.pt, r.grad_full, r.rs_stage, E, N, r.rank, L.S, L.flat, r.grad_shard, st);
  } else if (rs && !ce_rs) {
    for (Rank& r : L.ranks) launch_grad_reduce_scatter(r.pt, L.peers, E, r.rank, L.S, L.flat, r.grad_shard, st);
  }
  mark(L, st, kPhGradRS);
  if (deferred) join_rs(*deferred, st);  // long finished under this layer's GEMMs
  // join the planner stream (it finished long before the backward GEMMs did)
  if (L.planner_pending) CK(cudaStreamWaitEvent(st, L.ev_planned, 0));
}

Rank& rank_of(Layer& L, uint32_t vrank) {
  if (!L.virt) return L.ranks[0];
  if (vrank >= L.ranks.size()) throw Error(ErrorKind::invalid_argument, "vrank out of range");
  return L.ranks[vrank];
}

// Device-detected failures that have landed in the host-mapped words so far:
// report (MP_ERR_DEVICE, naming the causes) and clear them.  `bits` gets
// 1 << ErrWord for every set word.
uint32_t take_errors(Layer& L) {
  uint32_t bits = 0;
  for (int w = 0; w < kErrWords; ++w) {
    volatile unsigned* p = L.err_host + w;
    if (*p) bits |= 1u << w, *p = 0;
  }
  return bits;
}

void raise_errors(uint32_t bits) {
  if (!bits) return;
  std::string m = "FSEP layer step failed on the device:";
  if (bits & (1u << kErrRecvOverflow)) m += " receive buffer overflow (max_recv_rows too small; segments dropped);";
  if (bits & (1u << kErrBarrierTimeout)) m += " peer barrier timed out (a rank did not arrive);";
  if (bits & (1u << kErrRestoreTimeout)) m += " restored expert chunk never arrived (readiness flag timeout);";
  if (bits & (1u << kErrGuard)) m += " a kernel wrote past the end of a buffer (memory guard overwritten);";
  throw Error(ErrorKind::device, m);
}

// Device-detected failures (host-mapped words) and, on the NCCL transport, an
// asynchronous communicator failure (a peer gone, a network error) -> MP_ERR_DEVICE.
void poll_errors(Layer& L) {
  raise_errors(take_errors(L));
  if (L.nccl != nullptr) {
    ncclResult_t async = ncclSuccess;
    nccl_check(ncclCommGetAsyncError(L.nccl, &async), "ncclCommGetAsyncError");
    if (async != ncclSuccess && async != ncclInProgress) nccl_check(async, "NCCL communicator failed asynchronously");
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

using moeplan::capi::guarded;
using moeplan::capi::require;

extern "C" {

mp_status mp_fsep_layer_create(const mp_fsep_desc* desc, int device, mp_fsep_layer** out) {
  return guarded([&] {
    require(desc && out, "mp_fsep_layer_create: NULL argument");
    const mp_fsep_desc& d = *desc;
    require(d.world >= 1 && d.world <= static_cast<uint32_t>(kMaxRanks), "world must be in [1, 16]");
    require(d.n_experts >= 1 && d.n_experts <= static_cast<uint32_t>(kMaxExperts), "n_experts must be in [1, 256]");
    require(d.top_k >= 1 && d.top_k <= 8 && d.top_k <= d.n_experts, "top_k must be in [1, min(8, E)]");
    // hidden = 256 * CH for the token kernels' row widths (routing.cu FSEP_CH_SWITCH): 256 ... 8192,
    // e.g. 4096 (Mixtral), 2048, 5120, 6144, 7168 (DeepSeek-V3), 8192
    static constexpr int kHiddenCh[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 14, 16, 20, 24, 28, 32};
    require(d.hidden % 256 == 0 && std::find(std::begin(kHiddenCh), std::end(kHiddenCh),
                                             static_cast<int>(d.hidden / 256)) != std::end(kHiddenCh),
            "hidden must be 256 * {1-6, 8, 10, 12, 14, 16, 20, 24, 28, 32}");
    require(d.ffn % 128 == 0 && d.ffn > 0, "ffn must be a multiple of 128");
    require(d.capacity >= 1 && d.capacity <= d.n_experts && d.n_experts <= d.world * d.capacity,
            "capacity must satisfy 1 <= C <= E <= N*C");
    require(d.capacity <= 128, "capacity (experts per device) must be <= 128 (grouped-GEMM group table)");
    require(d.top_k <= d.capacity * d.world, "top_k too large");
    require(d.virtual_ranks || d.rank < d.world, "rank out of range");
    const long long flat = 3LL * d.hidden * d.ffn;
    require(flat % (8LL * d.world) == 0, "3*H*F must be divisible by 8*world (16-byte shard chunks)");
    auto L = std::make_unique<mp_fsep_layer>();
    L->d = d;
    L->device = device;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, device));
    L->N = static_cast<int>(d.world);
    L->E = static_cast<int>(d.n_experts);
    L->K = static_cast<int>(d.top_k);
    L->H = static_cast<int>(d.hidden);
    L->F = static_cast<int>(d.ffn);
    L->C = static_cast<int>(d.capacity);
    L->T_max = static_cast<int>(d.max_tokens);
    L->flat = flat;
    L->S = flat / L->N;
    L->virt = d.virtual_ranks != 0 || L->N == 1;
    L->resident = (d.flags & MP_FSEP_FLAG_RESIDENT_EXPERTS) != 0;
    L->local_first = (d.flags & MP_FSEP_FLAG_LOCAL_FIRST) != 0;
    L->defer_rs = (d.flags & MP_FSEP_FLAG_DEFER_RS) != 0;
    // de-duplicated token transfers pay off when a token has several slots per
    // device (top-k >= 4); FSEP_DEDUPE=0/1 overrides
    L->dedupe = L->N > 1 && d.top_k >= 4 && use_tma_dispatch();
    if (const char* v = std::getenv("FSEP_DEDUPE")) L->dedupe = L->N > 1 && std::string(v) != "0" && use_tma_dispatch();
    if (const char* v = std::getenv("FSEP_RESTORE_SPLIT")) L->restore_split = std::string(v) != "0";
    require(!L->resident || d.n_experts == d.world * d.capacity,
            "resident-expert (pure EP) mode needs E == N*C (one host per expert)");
    const long long worst = static_cast<long long>(d.max_tokens) * d.top_k * L->N + 128LL * L->C;
    L->cap = d.max_recv_rows ? static_cast<long long>(d.max_recv_rows) + 128LL * L->C : worst;
    require(L->cap < (1LL << 24), "receive rows must stay below 2^24");
    require(static_cast<long long>(d.max_tokens) * d.top_k < (1LL << kRowSrcShift), "max_tokens * top_k must stay below 2^26");
    // copy-engine communication for real multi-GPU mode (FSEP_COMM=kernel selects the SM kernels);
    // decided before carving the arena (push targets live in it; identical on every rank)
    // Virtual mode runs the same copy-engine transport between the emulated ranks with
    // MP_FSEP_FLAG_COPY_ENGINE (or FSEP_COMM=ce), so one GPU exercises the shipped N>1 path.
    const char* comm = std::getenv("FSEP_COMM");
    const bool want_ce = L->virt ? ((d.flags & MP_FSEP_FLAG_COPY_ENGINE) != 0 || (comm && std::string(comm) == "ce"))
                                 : !(comm && std::string(comm) == "kernel");
    L->ce_mode = L->N > 1 && want_ce && write_value_fn() != nullptr;
    require(!(L->virt && (d.flags & MP_FSEP_FLAG_COPY_ENGINE)) || L->ce_mode || L->N == 1,
            "copy-engine mode unavailable (cuStreamWriteValue32 entry point missing)");
    L->sm_push = L->ce_mode && comm && std::string(comm) == "sm";
    L->nccl_mode = !L->virt && L->N > 1 && comm && std::string(comm) == "nccl";
    if (L->nccl_mode) L->ce_mode = false;
    // SM push: one push kernel per restore, launched at the forward's start (while the SMs
    // are free), so its CTAs are resident before the persistent gate-up GEMM polls the
    // flags.  A second kernel launched after dispatch could not always get CTAs beside the
    // GEMM (flags then only landed after the readiness timeout) -- measured, Mixtral N=8.
    if (L->sm_push && !std::getenv("FSEP_RESTORE_SPLIT")) L->restore_split = false;
    // Two copy-engine lanes per peer when each restored chunk is large (Mixtral: 88 MB at
    // N=4; tokens/s +0.3 % at T=16384, +0.1 % at T=4096 over 3 alternations,
    // profiles/r02/ce_auto_lanes/); one for small chunks, where a second lane only adds
    // contention with the GEMMs (fine config, 4.3 MB chunks: -1.9 % / -3.3 %,
    // profiles/r02/n4_ce_lanes_*).
    L->ce_k = L->S * 2 >= (32ll << 20) ? 2 : 1;
    if (const char* v = std::getenv("FSEP_CE_STREAMS")) L->ce_k = std::clamp(std::atoi(v), 1, mp_fsep_layer::kMaxLanes);
    if (const char* v = std::getenv("FSEP_PUSH_CTAS")) L->push_ctas = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("FSEP_PUSH_PIECE_KB"))
      L->piece_bytes = static_cast<unsigned long long>(std::max(16, std::atoi(v))) * 1024ull;
    if (const char* v = std::getenv("FSEP_SPIN_TIMEOUT_MS"))
      L->spin_timeout_ns = static_cast<unsigned long long>(std::max(1.0, std::atof(v)) * 1e6);
    CK(cudaHostAlloc(&L->err_host, kErrWords * sizeof(unsigned), cudaHostAllocMapped));
    std::memset(L->err_host, 0, kErrWords * sizeof(unsigned));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&L->err_dev), L->err_host, 0));
    const int local = L->virt ? L->N : 1;
    L->ranks.resize(local);
    for (int v = 0; v < local; ++v) {
      L->ranks[v].rank = L->virt ? v : static_cast<int>(d.rank);
      allocate_rank(*L, L->ranks[v]);
    }
    finish_peers(*L);
    {
      std::vector<const unsigned char*> all;
      for (const Rank& r : L->ranks)
        for (const Guard& g : r.guards) all.push_back(g.at);
      L->n_guards = static_cast<int>(all.size());
      CK(cudaMalloc(&L->d_guards, all.size() * sizeof(void*)));
      CK(cudaMemcpy(L->d_guards, all.data(), all.size() * sizeof(void*), cudaMemcpyHostToDevice));
      CK(cudaMalloc(&L->d_guard_bad, sizeof(int)));
    }
    L->connected = L->virt;
    CK(cudaMallocHost(&L->layout_host, static_cast<size_t>(L->E) * L->N));
    CK(cudaMallocHost(&L->R_host, static_cast<size_t>(L->E) * L->N * 8));
    // default layout: even replication (sim.cpp:100-103 initial layout)
    require(mp_fsep_even_layout(L->N, L->E, L->C, L->layout_host) == MP_OK, "even layout failed");
    CK(cudaStreamCreateWithFlags(&L->side, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&L->plan_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&L->cap_stream, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&L->ev_fork, &L->ev_restored, &L->ev_hist, &L->ev_planned, &L->ev_rs_done, &L->ev_nccl_rs})
      CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    if (L->nccl_mode) CK(cudaMallocHost(&L->layout_ring, 4 * static_cast<size_t>(L->E) * L->N));
    for (auto& ring : L->ev_g)
      for (auto& e : ring) CK(cudaEventCreate(&e));
    if (const char* v = std::getenv("FSEP_PHASE_TIMING"); v && std::string(v) == "1") {
      L->phase_on = true;
      L->ev_p.resize(mp_fsep_layer::kPhaseRing);
      for (auto& ring : L->ev_p)
        for (auto& e : ring) CK(cudaEventCreate(&e));
      L->ev_ce_t.resize(mp_fsep_layer::kPhaseRing);
      for (auto& ring : L->ev_ce_t)
        for (auto& e : ring) CK(cudaEventCreate(&e));
    }
    if (const char* v = std::getenv("FSEP_RESTORE_BLOCKS")) L->restore_blocks = std::max(1, std::atoi(v));
    if (L->ce_mode) {
      for (int p = 0; p < L->N; ++p) {
        for (int j = 0; j < L->ce_k; ++j) {
          CK(cudaStreamCreateWithFlags(&L->ce[p * L->ce_k + j], cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&L->ev_ce[p * L->ce_k + j], cudaEventDisableTiming));
        }
      }
      CK(cudaEventCreateWithFlags(&L->ev_wg, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&L->ev_w2, cudaEventDisableTiming));
      CK(cudaMallocHost(&L->layout_ring, 4 * static_cast<size_t>(L->E) * L->N));
      if (L->sm_push) {
        L->task_cap = local * L->N * L->C;
        const size_t n = static_cast<size_t>(Layer::kTaskRing) * L->task_cap;
        CK(cudaMallocHost(&L->task_host, n * sizeof(CopyTask)));
        CK(cudaMalloc(&L->task_dev, n * sizeof(CopyTask)));
        CK(cudaMalloc(&L->done_dev, n * sizeof(unsigned)));
        for (auto& e : L->ev_task) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
    }
    CK(cudaMalloc(&L->d_peer_flags, sizeof(unsigned int*) * kMaxRanks));
    CK(cudaMalloc(&L->d_peer_rs_flags, sizeof(unsigned int*) * kMaxRanks));
    CK(cudaMalloc(&L->d_tok_table, sizeof(__nv_bfloat16*) * kMaxRanks));
    if (L->virt) {
      unsigned int* f[kMaxRanks] = {};
      for (int v = 0; v < local; ++v) f[v] = L->ranks[v].flags;
      CK(cudaMemcpy(L->d_peer_flags, f, sizeof(f), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(L->d_tok_table, L->peers.tok_rows, sizeof(L->peers.tok_rows), cudaMemcpyHostToDevice));
    }
    CK(cudaDeviceSynchronize());
    *out = L.release();
  });
}

void mp_fsep_layer_free(mp_fsep_layer* L) {
  if (!L) return;
  cudaSetDevice(L->device);
  if (L->prev && L->prev->next == L) L->prev->next = nullptr;
  if (L->next && L->next->prev == L) L->next->prev = nullptr;
  cudaDeviceSynchronize();
  if (L->graph) cudaGraphExecDestroy(L->graph);
  for (void* p : L->opened_ptrs) cudaIpcCloseMemHandle(p);
  for (Rank& r : L->ranks) {
    cudaFree(r.arena);
    cudaFree(r.priv);
  }
  cudaFree(L->d_peer_flags);
  cudaFree(L->d_peer_rs_flags);
  cudaFree(L->d_guards);
  cudaFree(L->d_guard_bad);
  cudaFree(L->d_tok_table);
  cudaFreeHost(L->layout_host);
  cudaFreeHost(L->R_host);
  cudaStreamDestroy(L->side);
  cudaStreamDestroy(L->plan_stream);
  cudaStreamDestroy(L->cap_stream);
  cudaFreeHost(L->err_host);
  if (L->ce_mode) {
    for (int p = 0; p < L->N; ++p) {
      for (int j = 0; j < L->ce_k; ++j) {
        cudaStreamDestroy(L->ce[p * L->ce_k + j]);
        cudaEventDestroy(L->ev_ce[p * L->ce_k + j]);
      }
    }
    cudaEventDestroy(L->ev_wg);
    cudaEventDestroy(L->ev_w2);
    cudaFreeHost(L->layout_ring);
    if (L->sm_push) {
      cudaFreeHost(L->task_host);
      cudaFree(L->task_dev);
      cudaFree(L->done_dev);
      for (auto e : L->ev_task) cudaEventDestroy(e);
    }
  }
  for (cudaEvent_t e : {L->ev_fork, L->ev_restored, L->ev_hist, L->ev_planned, L->ev_rs_done, L->ev_nccl_rs})
    cudaEventDestroy(e);
  if (L->nccl_mode) {
    cudaFreeHost(L->layout_ring);
    if (L->nccl) ncclCommDestroy(L->nccl);
  }
  for (auto& ring : L->ev_g)
    for (auto e : ring) cudaEventDestroy(e);
  for (auto& ring : L->ev_p)
    for (auto e : ring) cudaEventDestroy(e);
  for (auto& ring : L->ev_ce_t)
    for (auto e : ring) cudaEventDestroy(e);
  delete L;
}

size_t mp_fsep_ipc_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

mp_status mp_fsep_nccl_unique_id(void* out, size_t bytes) {
  return guarded([&] {
    require(out && bytes >= sizeof(ncclUniqueId), "mp_fsep_nccl_unique_id: buffer too small");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) throw Error(ErrorKind::device, "ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof(id));
  });
}

mp_status mp_fsep_layer_ipc_handle(mp_fsep_layer* L, void* out, size_t bytes) {
  return guarded([&] {
    require(L && out && bytes >= sizeof(cudaIpcMemHandle_t), "mp_fsep_layer_ipc_handle: bad argument");
    require(!L->virt, "ipc handles are only used in real multi-GPU mode");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, L->ranks[0].arena));
    std::memcpy(out, &h, sizeof(h));
  });
}

}  // extern "C"

namespace {
// Fills L's peer tables from every rank's arena base address (as mapped in this
// process); identical carving on every rank gives identical offsets.
void connect_bases(mp_fsep_layer* L, const std::vector<char*>& bases) {
  Rank& me = L->ranks[0];
  unsigned int* flags[kMaxRanks] = {};
  unsigned int* rs_flags[kMaxRanks] = {};
  auto off = [&](const void* q) { return static_cast<const char*>(q) - static_cast<char*>(me.arena); };
  for (int p = 0; p < L->N; ++p) {
    char* base = bases[static_cast<size_t>(p)];
    L->peers.x_rows[p] = reinterpret_cast<__nv_bfloat16*>(base + off(me.x_rows));
    L->peers.dy_rows[p] = reinterpret_cast<__nv_bfloat16*>(base + off(me.dy_rows));
    L->peers.tok_rows[p] = reinterpret_cast<__nv_bfloat16*>(base + off(me.tok_rows));
    L->peers.row_src[p] = reinterpret_cast<int*>(base + off(me.row_src));
    if (L->dedupe) {
      L->peers.stage[p] = reinterpret_cast<__nv_bfloat16*>(base + off(me.stage));
      L->peers.row_w[p] = reinterpret_cast<float*>(base + off(me.row_w));
    }
    if (L->ce_mode) {
      L->peer_restored[p] = reinterpret_cast<__nv_bfloat16*>(base + off(me.restored));
      L->peer_ready[p] = reinterpret_cast<unsigned*>(base + off(me.ready));
      L->peer_rs_stage[p] = reinterpret_cast<float*>(base + off(me.rs_stage));
    }
    L->peers.R_all[p] = reinterpret_cast<unsigned long long*>(base + off(me.R_all));
    L->peers.grad_full[p] = reinterpret_cast<float*>(base + off(me.grad_full));
    L->peers.shard[p] = reinterpret_cast<const __nv_bfloat16*>(base + off(me.shard));
    flags[p] = reinterpret_cast<unsigned int*>(base + off(me.flags));
    rs_flags[p] = reinterpret_cast<unsigned int*>(base + off(me.rs_flags));
  }
  CK(cudaMemcpy(L->d_peer_flags, flags, sizeof(flags), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(L->d_peer_rs_flags, rs_flags, sizeof(rs_flags), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(L->d_tok_table, L->peers.tok_rows, sizeof(L->peers.tok_rows), cudaMemcpyHostToDevice));
}
}  // namespace

extern "C" {

mp_status mp_fsep_layer_connect(mp_fsep_layer* L, const void* all_handles, const void* nccl_id) {
  return guarded([&] {
    require(L && all_handles, "mp_fsep_layer_connect: NULL argument");
    require(!L->virt, "connect is only used in real multi-GPU mode");
    CK(cudaSetDevice(L->device));
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(all_handles);
    std::vector<char*> bases(static_cast<size_t>(L->N));
    for (int p = 0; p < L->N; ++p) {
      if (p == L->ranks[0].rank) {
        bases[static_cast<size_t>(p)] = static_cast<char*>(L->ranks[0].arena);
      } else {
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
        L->opened_ptrs.push_back(ptr);
        bases[static_cast<size_t>(p)] = static_cast<char*>(ptr);
      }
    }
    connect_bases(L, bases);
    if (L->nccl_mode) {  // FSEP_COMM=nccl: one communicator per layer (collective over the ranks)
      require(nccl_id != nullptr, "mp_fsep_layer_connect: FSEP_COMM=nccl needs the NCCL unique id");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      nccl_check(ncclCommInitRank(&L->nccl, L->N, id, L->ranks[0].rank), "ncclCommInitRank");
    }
    L->connected = true;
  });
}

mp_status mp_fsep_layer_connect_local(mp_fsep_layer** layers, uint32_t n) {
  return guarded([&] {
    require(layers && n >= 1, "mp_fsep_layer_connect_local: bad argument");
    for (uint32_t i = 0; i < n; ++i) {
      require(layers[i] && !layers[i]->virt && layers[i]->N == static_cast<int>(n) &&
                  layers[i]->ranks[0].rank == static_cast<int>(i) && !layers[i]->nccl_mode,
              "mp_fsep_layer_connect_local: layers[i] must be real-mode rank i of an n-rank layer");
    }
    std::vector<char*> bases(n);
    for (uint32_t i = 0; i < n; ++i) bases[i] = static_cast<char*>(layers[i]->ranks[0].arena);
    for (uint32_t i = 0; i < n; ++i) {
      CK(cudaSetDevice(layers[i]->device));
      for (uint32_t j = 0; j < n; ++j) {
        if (layers[j]->device == layers[i]->device) continue;
        const cudaError_t e = cudaDeviceEnablePeerAccess(layers[j]->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CK(e);
      }
      connect_bases(layers[i], bases);
      layers[i]->connected = true;
    }
  });
}

mp_status mp_fsep_layer_load_expert(mp_fsep_layer* L, uint32_t expert, const void* w1, const void* w3, const void* w2,
                                    void* stream) {
  return guarded([&] {
    require(L && w1 && w3 && w2, "mp_fsep_layer_load_expert: NULL argument");
    require(expert < static_cast<uint32_t>(L->E), "expert out of range");
    CK(cudaSetDevice(L->device));
    L->restore_dirty = true;
    auto st = static_cast<cudaStream_t>(stream);
    const size_t n1 = static_cast<size_t>(L->F) * L->H;
    __nv_bfloat16 *tmp = nullptr, *flat = nullptr;
    CK(cudaMallocAsync(&tmp, 3 * n1 * 2, st));
    CK(cudaMallocAsync(&flat, 3 * n1 * 2, st));
    CK(cudaMemcpyAsync(tmp, w1, n1 * 2, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(tmp + n1, w3, n1 * 2, cudaMemcpyDefault, st));
    CK(cudaMemcpyAsync(tmp + 2 * n1, w2, n1 * 2, cudaMemcpyDefault, st));
    launch_pack_expert(tmp, tmp + n1, tmp + 2 * n1, L->H, L->F, flat, st);
    for (Rank& r : L->ranks)
      CK(cudaMemcpyAsync(r.shard + static_cast<long long>(expert) * L->S, flat + static_cast<long long>(r.rank) * L->S,
                         static_cast<size_t>(L->S) * 2, cudaMemcpyDeviceToDevice, st));
    CK(cudaFreeAsync(tmp, st));
    CK(cudaFreeAsync(flat, st));
  });
}

mp_status mp_fsep_layer_load_router(mp_fsep_layer* L, const void* wg, void* stream) {
  return guarded([&] {
    require(L && wg, "mp_fsep_layer_load_router: NULL argument");
    CK(cudaSetDevice(L->device));
    for (Rank& r : L->ranks)
      CK(cudaMemcpyAsync(r.wg, wg, static_cast<size_t>(L->E) * L->H * 2, cudaMemcpyDefault,
                         static_cast<cudaStream_t>(stream)));
  });
}

mp_status mp_fsep_layer_set_layout(mp_fsep_layer* L, const uint8_t* A) {
  return guarded([&] {
    require(L && A, "mp_fsep_layer_set_layout: NULL argument");
    // validate like validate_layout (types.cpp:103-113)
    for (int d = 0; d < L->N; ++d) {
      int held = 0;
      for (int e = 0; e < L->E; ++e) held += A[e * L->N + d] ? 1 : 0;
      require(held == L->C, "layout: every device must host exactly C experts");
    }
    for (int e = 0; e < L->E; ++e) {
      int reps = 0;
      for (int d = 0; d < L->N; ++d) reps += A[e * L->N + d] ? 1 : 0;
      require(reps >= 1, "layout: every expert needs a replica");
    }
    if (L->resident)
      for (int e = 0; e < L->E; ++e) {
        int reps = 0;
        for (int d = 0; d < L->N; ++d) reps += A[e * L->N + d] ? 1 : 0;
        require(reps == 1, "layout: resident-expert (pure EP) mode needs exactly one host per expert");
      }
    if (L->planner_pending) CK(cudaEventSynchronize(L->ev_planned));  // don't race the planner callback
    for (int i = 0; i < L->E * L->N; ++i) L->layout_host[i] = A[i] ? 1 : 0;
    L->restore_dirty = true;
  });
}

mp_status mp_fsep_layer_chain(mp_fsep_layer* L, mp_fsep_layer* next) {
  return guarded([&] {
    require(L, "mp_fsep_layer_chain: NULL layer");
    require(next != L, "mp_fsep_layer_chain: a layer cannot precede itself");
    require(!next || (next->N == L->N && next->device == L->device), "mp_fsep_layer_chain: layers must share devices");
    if (L->next && L->next->prev == L) {
      join_rs(*L->next, nullptr);  // nobody completes its deferred reduce-scatter any more
      L->next->prev = nullptr;
    }
    L->next = next;
    if (next) next->prev = L;
  });
}

mp_status mp_fsep_layer_attach_planner(mp_fsep_layer* L, mp_fsep_planner* planner) {
  return guarded([&] {
    require(L, "mp_fsep_layer_attach_planner: NULL layer");
    require(!(L->resident && planner), "resident-expert (pure EP) layers keep a fixed layout: no planner");
    if (L->planner_pending) CK(cudaEventSynchronize(L->ev_planned));
    L->planner = planner;
    L->planner_pending = false;
  });
}

mp_status mp_fsep_layer_forward(mp_fsep_layer* L, const void* x, const float* bias, uint32_t n_tokens, void* y,
                                void* stream) {
  return guarded([&] {
    const NvtxRange range("fsep.forward");
    require(L && x && y, "mp_fsep_layer_forward: NULL argument");
    require(L->connected, "mp_fsep_layer_forward: multi-GPU layer not connected");
    CK(cudaSetDevice(L->device));
    poll_errors(*L);
    L->launches_before = launches_issued();
    run_forward(*L, static_cast<const __nv_bfloat16*>(x), bias, static_cast<int>(n_tokens),
                static_cast<__nv_bfloat16*>(y), static_cast<cudaStream_t>(stream));
    CK(cudaGetLastError());
  });
}

mp_status mp_fsep_layer_backward(mp_fsep_layer* L, const void* dy, void* dx, void* stream) {
  return guarded([&] {
    const NvtxRange range("fsep.backward");
    require(L && dy && dx, "mp_fsep_layer_backward: NULL argument");
    CK(cudaSetDevice(L->device));
    poll_errors(*L);
    run_backward(*L, static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx),
                 static_cast<cudaStream_t>(stream));
    L->launches_step = launches_issued() - L->launches_before;
    ++L->step_no;
    CK(cudaGetLastError());
  });
}

mp_status mp_fsep_layer_histogram(mp_fsep_layer* L, uint64_t* R_out) {
  return guarded([&] {
    require(L && R_out, "mp_fsep_layer_histogram: NULL argument");
    CK(cudaEventSynchronize(L->ev_hist));
    std::memcpy(R_out, L->R_host, static_cast<size_t>(L->N) * L->E * 8);
  });
}

mp_status mp_fsep_layer_expert_grad(mp_fsep_layer* L, uint32_t expert, float* dw1, float* dw3, float* dw2,
                                    void* stream) {
  return guarded([&] {
    require(L && dw1 && dw3 && dw2, "mp_fsep_layer_expert_grad: NULL argument");
    require(expert < static_cast<uint32_t>(L->E), "expert out of range");
    require(is_device_ptr(dw1) && is_device_ptr(dw3) && is_device_ptr(dw2), "grad outputs must be device pointers");
    auto st = static_cast<cudaStream_t>(stream);
    join_rs(*L, st);  // a deferred reduce-scatter not yet completed by the previous layer
    if (L->resident && L->N > 1) {  // whole gradient on the expert's single host
      const uint8_t* A = L->cur_layout ? L->cur_layout : L->layout_host;
      for (Rank& r : L->ranks) {
        const std::vector<int> mine = hosted_experts(A, L->E, L->N, r.rank);
        const auto it = std::find(mine.begin(), mine.end(), static_cast<int>(expert));
        if (it == mine.end()) continue;
        launch_unpack_grad(r.grad_full + static_cast<long long>(it - mine.begin()) * L->flat, 0, L->flat, L->H, L->F,
                           dw1, dw3, dw2, st);
      }
      return;
    }
    for (Rank& r : L->ranks) {
      const long long lo = static_cast<long long>(r.rank) * L->S;
      launch_unpack_grad(r.grad_shard + static_cast<long long>(expert) * L->S, lo, lo + L->S, L->H, L->F, dw1, dw3,
                         dw2, st);
    }
  });
}

mp_status mp_fsep_layer_router_grad(mp_fsep_layer* L, uint32_t vrank, float* dwg, void* stream) {
  return guarded([&] {
    require(L && dwg, "mp_fsep_layer_router_grad: NULL argument");
    Rank& r = rank_of(*L, vrank);
    CK(cudaMemcpyAsync(dwg, r.dwg, static_cast<size_t>(L->E) * L->H * 4, cudaMemcpyDefault,
                       static_cast<cudaStream_t>(stream)));
  });
}

mp_status mp_fsep_layer_read(mp_fsep_layer* L, const char* name, uint32_t vrank, void* dst, uint64_t bytes,
                             uint64_t* needed) {
  return guarded([&] {
    require(L && name, "mp_fsep_layer_read: NULL argument");
    Rank& r = rank_of(*L, vrank);
    const std::string n(name);
    const size_t T = static_cast<size_t>(L->T_step), K = L->K, E = L->E, N = L->N, H = L->H, F = L->F, C = L->C;
    const size_t cap = static_cast<size_t>(L->cap);
    const void* src = nullptr;
    size_t sz = 0;
    if (n == "topk_idx") src = r.topk_idx, sz = T * K * 4;
    else if (n == "topk_w") src = r.topk_w, sz = T * K * 4;
    else if (n == "slot_dst") src = r.slot_dst, sz = T * K * 4;
    else if (n == "dl") src = r.dl, sz = T * K * 4;
    else if (n == "R") src = r.R_all, sz = N * E * 8;
    else if (n == "layout") src = r.layout_dev, sz = E * N;
    else if (n == "seg_rows") src = r.pt->seg_rows, sz = C * 4;
    else if (n == "seg_off") src = r.pt->seg_off, sz = C * 4;
    else if (n == "slot_expert") src = r.pt->slot_expert, sz = C * 4;
    else if (n == "status") src = &r.pt->status, sz = 4;
    else if (n == "total_rows") src = &r.pt->total_rows, sz = 4;
    else if (n == "x_rows") src = r.x_rows, sz = cap * H * 2;
    else if (n == "dy_rows") src = r.dy_rows, sz = cap * H * 2;
    else if (n == "tok_rows") src = r.tok_rows, sz = T * K * H * 2;
    else if (n == "row_src") src = r.row_src, sz = cap * 4;
    else if (n == "h") src = r.h, sz = cap * 2 * F * 2;
    else if (n == "act") src = r.act, sz = cap * F * 2;
    else if (n == "restored") src = r.restored, sz = C * static_cast<size_t>(L->flat) * 2;
    else if (n == "grad_full") src = r.grad_full, sz = C * static_cast<size_t>(L->flat) * 4;
    else if (n == "barrier_status") src = r.flags + N, sz = 4;
    else if (n == "ready" && r.ready) src = r.ready, sz = C * N * 4;  // readiness flags [slot][source]
    else if (n == "restore_epoch") src = &L->restore_epoch, sz = 4;
    else throw Error(ErrorKind::invalid_argument, "mp_fsep_layer_read: unknown buffer " + n);
    if (needed) *needed = sz;
    if (dst) {
      require(bytes >= sz, "mp_fsep_layer_read: destination too small");
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(dst, src, sz, cudaMemcpyDefault));
    }
  });
}

mp_status mp_fsep_layer_stats(mp_fsep_layer* L, uint64_t* kernel_launches, double* gemm_ms, double* gemm_flops) {
  return guarded([&] {
    require(L, "mp_fsep_layer_stats: NULL layer");
    // Average over the steps completed since the last reset (at most the ring size).
    const long long n = std::min<long long>(L->step_no - L->stats_from, Layer::kRing);
    require(n > 0, "mp_fsep_layer_stats: no completed step since reset");
    double ms = 0.0;
    for (long long s = L->step_no - n; s < L->step_no; ++s) {
      cudaEvent_t* ev = L->ev_g[s % Layer::kRing];
      CK(cudaEventSynchronize(ev[3]));
      float f0 = 0, f1 = 0;
      CK(cudaEventElapsedTime(&f0, ev[0], ev[1]));
      CK(cudaEventElapsedTime(&f1, ev[2], ev[3]));
      ms += static_cast<double>(f0) + static_cast<double>(f1);
    }
    if (kernel_launches) *kernel_launches = L->launches_step;
    if (gemm_ms) *gemm_ms = ms / static_cast<double>(n);
    if (gemm_flops) {
      // algorithmic FLOPs of this rank's grouped GEMMs per step: 18*H*F per token-slot computed here
      // (fwd 6HF + bwd 12HF), counted from the device's segment sizes of the last step
      unsigned long long rows = 0;
      for (Rank& r : L->ranks) {
        std::vector<int> seg(static_cast<size_t>(L->C));
        CK(cudaMemcpy(seg.data(), r.pt->seg_rows, seg.size() * 4, cudaMemcpyDeviceToHost));
        for (int v : seg) rows += static_cast<unsigned long long>(v);
      }
      *gemm_flops = 18.0 * L->H * L->F * static_cast<double>(rows);
    }
    poll_errors(*L);  // the step whose numbers these are must not have failed
  });
}

mp_status mp_fsep_layer_check(mp_fsep_layer* L, uint32_t* bits) {
  if (bits) *bits = 0;
  return guarded([&] {
    require(L, "mp_fsep_layer_check: NULL layer");
    CK(cudaSetDevice(L->device));
    CK(cudaDeviceSynchronize());
    uint32_t b = take_errors(*L);
    // memory guards after every buffer of every local rank (the memcheck stand-in)
    std::string guard_msg;
    if (L->n_guards > 0) {
      const int none = 0x7fffffff;
      CK(cudaMemcpy(L->d_guard_bad, &none, sizeof(int), cudaMemcpyHostToDevice));
      launch_guard_check(L->d_guards, L->n_guards, kGuardByte, L->d_guard_bad, nullptr);
      int bad = none;
      CK(cudaMemcpy(&bad, L->d_guard_bad, sizeof(int), cudaMemcpyDeviceToHost));
      if (bad != none) {
        b |= 1u << kErrGuard;
        int idx = bad;
        for (const Rank& r : L->ranks) {
          if (idx < static_cast<int>(r.guards.size())) {
            guard_msg = std::string(" (guard after '") + r.guards[static_cast<size_t>(idx)].after + "' of rank " +
                        std::to_string(r.rank) + ")";
            break;
          }
          idx -= static_cast<int>(r.guards.size());
        }
      }
    }
    if (bits) *bits = b;
    try {
      raise_errors(b);
    } catch (const Error& e) {
      throw Error(ErrorKind::device, std::string(e.what()) + guard_msg);
    }
  });
}

// Transport probe (dev/bench): `iters` full shard restores of the current layout
// (barrier, pushes of every slot, join of this rank's pushes, barrier), timed with
// events on the layer's capture stream.  *ms = mean per restore.
mp_status mp_fsep_layer_debug_restore(mp_fsep_layer* L, int iters, double* ms) {
  return guarded([&] {
    require(L && ms && iters > 0, "mp_fsep_layer_debug_restore: bad argument");
    require(L->ce_mode, "mp_fsep_layer_debug_restore: push transport (copy engines / SM push) only");
    CK(cudaSetDevice(L->device));
    cudaStream_t st = L->cap_stream;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    snapshot_layout(*L, st);
    barrier(*L, st);
    CK(cudaEventRecord(a, st));
    for (int i = 0; i < iters; ++i) {
      push_restore(*L, st);
      for (int p = 0; p < L->lanes(); ++p) CK(cudaStreamWaitEvent(st, L->ev_ce[p], 0));
      barrier(*L, st);
    }
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, a, b));
    *ms = static_cast<double>(t) / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    poll_errors(*L);
  });
}

mp_status mp_fsep_layer_debug_inject(mp_fsep_layer* L, const char* what) {
  return guarded([&] {
    require(L && what, "mp_fsep_layer_debug_inject: NULL argument");
    CK(cudaSetDevice(L->device));
    const std::string w(what);
    if (w == "drop_restore_flag") {
      require(L->ce_mode, "drop_restore_flag needs copy-engine mode");
      L->drop_flag = L->virt ? 1 : L->ranks[0].rank;  // virtual: emulated rank 1's push to a peer
    } else if (w == "clear_errors") {  // drop the landed error words without reporting (profiling probes)
      take_errors(*L);
    } else if (w == "overwrite_guard") {  // a one-byte overrun past x_rows of the first local rank
      const Guard& g = L->ranks[0].guards.front();
      CK(cudaMemset(const_cast<unsigned char*>(g.at), 0, 1));
    } else if (w == "barrier_timeout") {
      require(L->virt && L->N > 1, "barrier_timeout is emulated in virtual mode (rank 0 waits alone)");
      launch_peer_barrier(L->d_peer_flags, L->N, 0, L->epoch + 0x40000000u, L->err_dev, L->spin_timeout_ns, nullptr);
      CK(cudaDeviceSynchronize());
    } else {
      throw Error(ErrorKind::invalid_argument, "mp_fsep_layer_debug_inject: unknown condition " + w);
    }
  });
}

mp_status mp_fsep_layer_phase_ms(mp_fsep_layer* L, double* out, uint32_t n) {
  return guarded([&] {
    require(L && out, "mp_fsep_layer_phase_ms: NULL argument");
    require(L->phase_on, "phase timing is off (set FSEP_PHASE_TIMING=1 before creating the layer)");
    require(n >= static_cast<uint32_t>(kPhCount), "mp_fsep_layer_phase_ms: need kPhCount outputs");
    const long long cnt = std::min<long long>(L->step_no - L->stats_from, mp_fsep_layer::kPhaseRing);
    require(cnt > 0, "mp_fsep_layer_phase_ms: no completed step since reset");
    std::vector<double> acc(kPhCount, 0.0);
    const bool restore = L->N > 1 && !L->resident;
    for (long long s = L->step_no - cnt; s < L->step_no; ++s) {
      auto& ev = L->ev_p[static_cast<size_t>(s % mp_fsep_layer::kPhaseRing)];
      CK(cudaEventSynchronize(ev[kPhGradRS]));
      // out[i] (i < kPhGradRS) = time from mark i to mark i+1 on the main stream
      for (int i = kPhFwdBegin; i < kPhGradRS; ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ev[i], ev[i + 1]) == cudaSuccess) acc[i] += ms;
      }
      float tot = 0.f;
      if (cudaEventElapsedTime(&tot, ev[kPhFwdBegin], ev[kPhGradRS]) == cudaSuccess) acc[kPhGradRS] += tot;
      if (restore) {
        float a = 0.f, b = 0.f;
        if (cudaEventElapsedTime(&a, ev[kPhFwdBegin], ev[kPhRestoreBegin]) == cudaSuccess) acc[kPhRestoreBegin] += a;
        if (cudaEventElapsedTime(&b, ev[kPhRestoreBegin], ev[kPhRestoreEnd]) == cudaSuccess) acc[kPhRestoreEnd] += b;
      }
      cudaGetLastError();
    }
    // out[kPhStepBegin]: top of the forward -> first phase mark (layout snapshot / H2D);
    // out[kPhCount]: previous step's end -> this step's top (idle gap between steps);
    // out[kPhCount + 1]: host time blocked on the planner per step
    double gap = 0.0;
    long long ngap = 0;
    for (long long s = L->step_no - cnt; s < L->step_no; ++s) {
      auto& ev = L->ev_p[static_cast<size_t>(s % mp_fsep_layer::kPhaseRing)];
      float a = 0.f;
      if (cudaEventElapsedTime(&a, ev[kPhStepBegin], ev[kPhFwdBegin]) == cudaSuccess) acc[kPhStepBegin] += a;
      if (s > L->stats_from) {
        auto& pv = L->ev_p[static_cast<size_t>((s - 1) % mp_fsep_layer::kPhaseRing)];
        if (cudaEventElapsedTime(&a, pv[kPhGradRS], ev[kPhStepBegin]) == cudaSuccess) gap += a, ++ngap;
      }
      cudaGetLastError();
    }
    for (int i = 0; i < kPhCount; ++i) out[i] = acc[static_cast<size_t>(i)] / static_cast<double>(cnt);
    if (n > static_cast<uint32_t>(kPhCount)) out[kPhCount] = ngap ? gap / static_cast<double>(ngap) : 0.0;
    if (n > static_cast<uint32_t>(kPhCount) + 1) out[kPhCount + 1] = L->host_wait_ms / static_cast<double>(cnt);
    // out[kPhCount + 4]: restore begin -> last copy-engine push landed (copy-engine mode)
    if (n > static_cast<uint32_t>(kPhCount) + 4) {
      double land = 0.0;
      long long nl = 0;
      for (long long s = L->step_no - cnt; s < L->step_no && L->ce_mode && restore; ++s) {
        auto& ev = L->ev_p[static_cast<size_t>(s % mp_fsep_layer::kPhaseRing)];
        auto& ce = L->ev_ce_t[static_cast<size_t>(s % mp_fsep_layer::kPhaseRing)];
        float mx = 0.f;
        bool ok = false;
        for (int d = 0; d < L->N; ++d) {
          if (d == L->ranks[0].rank) continue;
          float a = 0.f;
          if (cudaEventElapsedTime(&a, ev[kPhRestoreBegin], ce[d]) == cudaSuccess) mx = std::max(mx, a), ok = true;
        }
        cudaGetLastError();
        if (ok) land += mx, ++nl;
      }
      out[kPhCount + 4] = nl ? land / static_cast<double>(nl) : 0.0;
    }
    // out[kPhCount + 2 / + 3]: forward top -> R on the host / -> planner callback done
    if (n > static_cast<uint32_t>(kPhCount) + 3) {
      double h = 0.0, pl = 0.0;
      for (long long s = L->step_no - cnt; s < L->step_no; ++s) {
        auto& ev = L->ev_p[static_cast<size_t>(s % mp_fsep_layer::kPhaseRing)];
        float a = 0.f;
        if (cudaEventElapsedTime(&a, ev[kPhStepBegin], ev[kPhHistD2H]) == cudaSuccess) h += a;
        if (L->planner && cudaEventElapsedTime(&a, ev[kPhStepBegin], ev[kPhPlanned]) == cudaSuccess) pl += a;
        cudaGetLastError();
      }
      out[kPhCount + 2] = h / static_cast<double>(cnt);
      out[kPhCount + 3] = pl / static_cast<double>(cnt);
    }
  });
}

mp_status mp_fsep_layer_stats_reset(mp_fsep_layer* L) {
  return guarded([&] {
    require(L, "mp_fsep_layer_stats_reset: NULL layer");
    L->stats_from = L->step_no;
    L->host_wait_ms = 0.0;
  });
}

mp_status mp_fsep_layer_graph_step(mp_fsep_layer* L, const void* x, const float* bias, uint32_t n_tokens, void* y,
                                   const void* dy, void* dx, void* stream) {
  return guarded([&] {
    const NvtxRange range("fsep.graph_step");
    require(L && x && y && dy && dx, "mp_fsep_layer_graph_step: NULL argument");
    auto st = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(L->device));
    poll_errors(*L);
    const void* key[5] = {x, bias, y, dy, dx};
    const bool same = L->graph && std::memcmp(key, L->graph_key, sizeof(key)) == 0 && L->T_step == static_cast<int>(n_tokens);
    if (!same) {
      if (L->graph) cudaGraphExecDestroy(L->graph);
      L->graph = nullptr;
      cudaGraph_t g;
      // Capture on the layer's own stream (the caller's may be the legacy default
      // stream, which cannot be captured).  Events from eager steps cannot be waited
      // on inside a capture: settle the planner first.
      if (L->planner_pending) CK(cudaEventSynchronize(L->ev_planned));
      L->planner_pending = false;
      // A captured graph must not bake layout-dependent copy addresses: graphs use
      // the device-side (layout read on the GPU) restore / reduce-scatter kernels.
      const bool ce_saved = L->ce_mode, nccl_saved = L->nccl_mode;
      L->ce_mode = false;
      L->nccl_mode = false;
      struct Restore {
        mp_fsep_layer* l;
        bool ce, nccl;
        ~Restore() {
          l->ce_mode = ce;
          l->nccl_mode = nccl;
        }
      } restore_ce{L, ce_saved, nccl_saved};
      cudaStream_t cs = L->cap_stream;
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      const uint64_t l0 = launches_issued();
      try {
        run_forward(*L, static_cast<const __nv_bfloat16*>(x), bias, static_cast<int>(n_tokens),
                    static_cast<__nv_bfloat16*>(y), cs);
        run_backward(*L, static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx), cs);
      } catch (...) {
        cudaStreamEndCapture(cs, &g);
        throw;
      }
      L->launches_step = launches_issued() - l0;
      CK(cudaStreamEndCapture(cs, &g));
      CK(cudaGraphInstantiate(&L->graph, g, 0));
      CK(cudaGraphDestroy(g));
      std::memcpy(L->graph_key, key, sizeof(key));
    }
    CK(cudaGraphLaunch(L->graph, st));
    // the graph joins its planner node internally; its event records are capture-internal
    L->planner_pending = false;
  });
}

}  // extern "C"
