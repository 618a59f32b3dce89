/* B200 FSEP framework -- C ABI of the FSEP MoE-layer step (GPU) and of the
 * array-level planner entry points it uses every step.
 *
 * The reference (/root/reference/proj) stops at the planner: its C ABI
 * (moeplan.h) emits layouts and routing plans as JSON for one trace layer
 * (mp_plan_layer_json, /root/reference/proj/src/capi.cpp:218-226 ->
 * commands.cpp:32-100).  A runtime needs the same computation on raw arrays,
 * once per (layer, step), without JSON; and it needs the GPU layer step that
 * consumes the result.  These entry points add exactly that, under the same
 * conventions as moeplan.h (mp_status returns, thread-local mp_last_error,
 * opaque caller-owned handles, no exceptions across the ABI, plain pointers and
 * sizes only -- no torch types).
 *
 * Layout of the arrays crossing this boundary (all row-major):
 *   R  [N][E]  uint64  token-slot counts, row i = source device i   (RoutingMatrix, types.hpp:26-52)
 *   A  [E][N]  uint8   0/1 replica placement                        (ExpertLayout,  types.hpp:63-87)
 *   S  [N][E][N] uint64 tokens (src, expert, dst)                   (RoutingPlan,   types.hpp:91-106, dense)
 *
 * GPU-side tensors (device pointers unless noted; bf16 = IEEE bfloat16 bits):
 *   x, y, dy, dx   [T][H] bf16 per rank (virtual mode: the ranks' blocks are concatenated)
 *   bias           [T][E] fp32 per rank, added to the router logits (routing-skew injection; may be NULL)
 *   expert weights: w1 (gate) [F][H], w3 (up) [F][H], w2 (down) [H][F] bf16 per expert
 *   router weight : wg [E][H] bf16
 * All GPU calls take a cudaStream_t (passed as void*) and are asynchronous
 * with respect to the host unless stated otherwise.
 */
#ifndef MOEPLAN_FSEP_H_
#define MOEPLAN_FSEP_H_

#include <stddef.h>
#include <stdint.h>

#include "moeplan.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ======================= array-level planner ============================== */

typedef struct mp_fsep_planner mp_fsep_planner;

/* A per-layer planner with history, following the runtime's one-iteration lag
 * (/root/reference/proj/src/sim.cpp:99-149): the layout for step t is
 * plan_layout(R_0..R_{t-1}) with the layer-salted seed
 * mix_seed(seed, "layr", layer) (sim.cpp:108-109).  Uses the config's topology,
 * cost, model.capacity and planner blocks (config.cpp:85-178). */
mp_status mp_fsep_planner_create(const mp_config* config, uint32_t n_devices, uint32_t layer,
                                 mp_fsep_planner** out);
/* Append one observed R (host array, N*E uint64) to the history. */
mp_status mp_fsep_planner_observe(mp_fsep_planner* planner, const uint64_t* R);
/* Layout for the next step: plan_layout over the history (planner.cpp:369-414),
 * or the even-replication layout when the history is empty (sim.cpp:100-103). */
mp_status mp_fsep_planner_next(mp_fsep_planner* planner, uint8_t* A_out);
void mp_fsep_planner_free(mp_fsep_planner* planner);

/* SURVEY 8(b)'s mp_fsep_plan_next: the layout for the next step of MoE layer `layer`
 * from one observed R (history = [R]) with the config's topology / cost / capacity /
 * planner blocks and the layer-salted seed -- array I/O, no JSON; equals the layout
 * mp_plan_layer_json reports after an iteration with this R in "last" history mode. */
mp_status mp_fsep_plan_next(const mp_config* config, const uint64_t* R, uint32_t n_devices, uint32_t layer,
                            uint8_t* A_out);

/* One-shot plan_layout on a single R (history = [R]) -- the hot call timed in
 * the CPU baseline. seed is used as-is (no layer salting). */
mp_status mp_fsep_plan_layout(uint32_t n_devices, uint32_t n_experts, uint32_t capacity, double bandwidth,
                              double v_comm, double v_comp, double b_comp, uint32_t epsilon, uint64_t seed,
                              const uint64_t* R, uint8_t* A_out);
/* lite_routing (planner.cpp:238-287) on a single-node topology, dense S output. */
mp_status mp_fsep_lite_routing(uint32_t n_devices, uint32_t n_experts, const uint64_t* R, const uint8_t* A,
                               uint64_t* S_out);
/* static_ep_layout (planner.cpp:289-296) / even_replication_layout (:298-307). */
mp_status mp_fsep_static_layout(uint32_t n_devices, uint32_t n_experts, uint32_t capacity, uint8_t* A_out);
mp_status mp_fsep_even_layout(uint32_t n_devices, uint32_t n_experts, uint32_t capacity, uint8_t* A_out);
/* time_cost (cost.cpp:39-73) of lite_routing(R, A) on Topology(1, N, bw, bw). */
mp_status mp_fsep_time_cost(uint32_t n_devices, uint32_t n_experts, const uint64_t* R, const uint8_t* A,
                            double bandwidth, double v_comm, double v_comp, double b_comp, double* t_comm,
                            double* t_comp, double* t_total, uint64_t* max_recv);

/* Expert popularity of the synthetic drifting trace (generate_trace semantics,
 * trace.cpp:89-129) before integer rounding: out[layer][iteration][expert]
 * (doubles, n_layers*n_iterations*n_experts).  spec_json as mp_trace_generate.
 * Drives the routing bias of the multi-layer dynamic-skew benchmark. */
mp_status mp_fsep_trace_popularity(const char* spec_json, double* out, uint64_t capacity);

/* Trace export: build an mp_trace from observed histograms (e.g. every step's
 * mp_fsep_layer_histogram) and write it with mp_trace_save in the reference
 * JSONL format {"iter","layer","R"} (trace.cpp:220-235), so the reference
 * tooling (mp_simulate / mp_plan_layer_json / moeplan simulate) replays real
 * B200 routing.  Records must be unique per (iter, layer). */
mp_status mp_fsep_trace_create(uint32_t n_devices, uint32_t n_experts, mp_trace** out);
mp_status mp_fsep_trace_append(mp_trace* trace, uint32_t iteration, uint32_t layer, const uint64_t* R);

/* ========================= GPU FSEP layer step ============================= */

typedef struct mp_fsep_layer mp_fsep_layer;

typedef struct mp_fsep_desc {
  uint32_t n_experts;     /* E */
  uint32_t top_k;         /* K */
  uint32_t hidden;        /* H  (multiple of 256) */
  uint32_t ffn;           /* F  per-expert SwiGLU width (multiple of 128) */
  uint32_t max_tokens;    /* T  tokens per rank per step (upper bound) */
  uint32_t capacity;      /* C  experts materialised per device (K <= C <= E, E <= N*C) */
  uint32_t world;         /* N  ranks */
  uint32_t rank;          /* this process's rank (real mode) */
  uint32_t virtual_ranks; /* 0 = real mode (one process per GPU, N processes);
                             1 = all N ranks emulated on this GPU (tests/correctness) */
  uint32_t flags;         /* MP_FSEP_FLAG_* bits, 0 = FSEP (restore + reduce-scatter every step) */
  uint64_t max_recv_rows; /* receive-buffer rows per rank; 0 = worst case T*K*N */
} mp_fsep_desc;

/* Pure expert parallelism (the baseline FSEP is compared against): every expert
 * has exactly one host (E == N*C, fixed layout via mp_fsep_layer_set_layout, no
 * planner), hosted experts stay restored across steps (re-restored only after
 * set_layout / load_expert) and expert gradients stay whole on their host (no
 * reduce-scatter); mp_fsep_layer_expert_grad then returns the gradient of
 * experts hosted by this process's rank(s) and leaves the outputs untouched for
 * the others. */
#define MP_FSEP_FLAG_RESIDENT_EXPERTS 1u
/* Local-first token routing (NOT the reference's lite_routing, planner.cpp:238-287;
 * opt-in, labelled non-parity): a source rank that hosts a replica of expert e
 * keeps all of its e-tokens local; other sources split their e-tokens over e's
 * replicas by lite routing's share/remainder rule.  Cuts NVLink token traffic on
 * one NVSwitch node; replica loads stay near-balanced when ranks see similar
 * routing distributions. */
#define MP_FSEP_FLAG_LOCAL_FIRST 2u
/* Virtual mode only: run the real multi-GPU transport between the emulated
 * ranks -- copy-engine shard-restore pushes, each followed by a
 * cuStreamWriteValue32 readiness flag polled per (slot, source) by the gate-up
 * GEMM's producer, copy-engine gradient pushes into the owners' staging rows and
 * the owner-side ascending-device sum -- instead of the device-side restore /
 * reduce-scatter kernels.  This is how one GPU checks the shipped N>1 data plane
 * against the oracle (real mode always uses it unless FSEP_COMM=kernel). */
#define MP_FSEP_FLAG_COPY_ENGINE 4u
/* Gradient-communication delay (PAPER Fig.5(e)): for a layer with a
 * chained predecessor (mp_fsep_layer_chain(prev, layer)), the owner-side half of
 * this layer's gradient reduce-scatter -- waiting for the replicas' pushed chunks,
 * the cross-rank barrier and the ascending-device sum -- is not run at the end of
 * this layer's backward but on a side stream under the predecessor's backward
 * GEMMs (the next expert layer in backward order).  Copy-engine mode only.  The
 * gradients are final once the predecessor's backward has run, or on the stream
 * passed to mp_fsep_layer_expert_grad (which completes a still-pending deferral). */
#define MP_FSEP_FLAG_DEFER_RS 8u

mp_status mp_fsep_layer_create(const mp_fsep_desc* desc, int device, mp_fsep_layer** out);
void mp_fsep_layer_free(mp_fsep_layer* layer);

/* Real multi-GPU mode only.  Exchange protocol (any transport, e.g.
 * torch.distributed all_gather on the bytes):
 *   1. every rank: mp_fsep_layer_ipc_handle -> blob of mp_fsep_ipc_bytes() bytes
 *   2. all-gather the N blobs (rank order); rank 0 also makes an NCCL id with
 *      mp_fsep_nccl_unique_id and broadcasts it
 *   3. every rank: mp_fsep_layer_connect(all blobs, nccl id)              */
size_t mp_fsep_ipc_bytes(void);
mp_status mp_fsep_nccl_unique_id(void* out, size_t bytes);
mp_status mp_fsep_layer_ipc_handle(mp_fsep_layer* layer, void* out, size_t bytes);
mp_status mp_fsep_layer_connect(mp_fsep_layer* layer, const void* all_handles, const void* nccl_id);
/* One process driving all N GPUs (tools, profiling): connect real-mode layers
 * layers[i] = rank i (each created on its own device) through direct peer access
 * instead of CUDA IPC. */
mp_status mp_fsep_layer_connect_local(mp_fsep_layer** layers, uint32_t n);

/* Parameters.  Weights are given unfused and unsharded (device or pinned host
 * pointers); each rank keeps its 1/N FSEP shard of every expert.  vrank
 * selects the emulated rank in virtual mode (ignored in real mode). */
mp_status mp_fsep_layer_load_expert(mp_fsep_layer* layer, uint32_t expert, const void* w1, const void* w3,
                                    const void* w2, void* stream);
mp_status mp_fsep_layer_load_router(mp_fsep_layer* layer, const void* wg, void* stream);

/* Expert layout for the NEXT forward (host array E*N).  The shard restore for
 * it is issued at the next forward (copy-engine pushes in real multi-GPU mode,
 * a restore kernel on a side stream in virtual mode). */
mp_status mp_fsep_layer_set_layout(mp_fsep_layer* layer, const uint8_t* A);

/* Attach a planner (mp_fsep_planner_create): after every forward's router the
 * runtime copies R to pinned host memory on a side stream and runs
 * observe(R) + next() in a stream host callback, so the layout of step t+1 is
 * planned from R_t while step t's GEMMs run (one-iteration lag, sim.cpp:114-131),
 * with no host synchronisation.  NULL detaches.  The planner must outlive the
 * layer or be detached first. */
mp_status mp_fsep_layer_attach_planner(mp_fsep_layer* layer, mp_fsep_planner* planner);

/* Layer chaining (PAPER Fig.5 schedule): after `layer`'s gate-up GEMM in each forward,
 * the shard restore of `next` (the next MoE layer, same devices) is issued on
 * next's copy engines, so it overlaps `layer`'s expert MLP; next's forward then
 * skips its own restore.  Copy-engine mode (real multi-GPU) only; NULL unchains.
 * Both layers' forwards must run every step in order (layer, then next). */
mp_status mp_fsep_layer_chain(mp_fsep_layer* layer, mp_fsep_layer* next);

/* Forward / backward of one step.  n_tokens <= max_tokens (per rank). */
mp_status mp_fsep_layer_forward(mp_fsep_layer* layer, const void* x, const float* bias, uint32_t n_tokens,
                                void* y, void* stream);
mp_status mp_fsep_layer_backward(mp_fsep_layer* layer, const void* dy, void* dx, void* stream);

/* R observed by the last forward (host array N*E); synchronises with the
 * forward's histogram event only (not with the whole step). */
mp_status mp_fsep_layer_histogram(mp_fsep_layer* layer, uint64_t* R_out);

/* Gradients after backward.  Expert grads are gathered from the fp32 shards
 * into full unfused fp32 tensors dw1/dw3 [F][H], dw2 [H][F] (device or host
 * pointers); router grad dwg [E][H] fp32 (sum over this rank's tokens). */
mp_status mp_fsep_layer_expert_grad(mp_fsep_layer* layer, uint32_t expert, float* dw1, float* dw3, float* dw2,
                                    void* stream);
mp_status mp_fsep_layer_router_grad(mp_fsep_layer* layer, uint32_t vrank, float* dwg, void* stream);

/* Test/inspection export of a named internal buffer of rank `vrank` into dst
 * (device or host).  If dst is NULL only *needed is written.  Names:
 *   "topk_idx" i32[T][K], "topk_w" f32[T][K], "slot_dst" u32[T][K] (dst<<24|row),
 *   "dl" f32[T][K], "R" u64[N][E], "layout" u8[E][N], "seg_rows" i32[C],
 *   "seg_off" i32[C], "slot_expert" i32[C], "total_rows" i32, "status" i32
 *   (1 = receive-buffer overflow: segments dropped, step invalid),
 *   "x_rows" / "dy_rows" bf16[cap][H], "row_src" i32[cap] (src<<26 | t*K+k, -1 pad),
 *   "tok_rows" bf16[T*K][H] (this rank's slot rows: y after forward, dX after
 *   backward), "h" bf16[cap][2F] (interleaved gate/up 128-col blocks),
 *   "act" bf16[cap][F], "restored" bf16[C][3HF], "grad_full" f32[C][3HF],
 *   "barrier_status" u32 (nonzero: a peer barrier timed out)                    */
mp_status mp_fsep_layer_read(mp_fsep_layer* layer, const char* name, uint32_t vrank, void* dst, uint64_t bytes,
                             uint64_t* needed);

/* Kernel launches of the last forward+backward; mean CUDA-event time per step
 * of the grouped-GEMM class (the dominant kernels) over the steps since
 * mp_fsep_layer_stats_reset, and their algorithmic FLOPs per step (18*H*F per
 * token-slot computed on this rank).  Used by bench.py's roofline line. */
mp_status mp_fsep_layer_stats(mp_fsep_layer* layer, uint64_t* kernel_launches, double* gemm_ms, double* gemm_flops);
mp_status mp_fsep_layer_stats_reset(mp_fsep_layer* layer);
/* Per-phase mean times (ms) since the last reset, when the layer was created with
 * FSEP_PHASE_TIMING=1 in the environment.  out[0..18]: consecutive main-stream
 * phases (param barrier, router+scan, R barrier, plan, dispatch, dispatch barrier
 * (+ expansion), restore wait, gate-up GEMM, down GEMM, barrier, combine,
 * combine-bwd + router wgrad, barrier (+ expansion), bwd GEMMs, wait for own
 * reduce-scatter pushes, barrier, reduce-scatter sum, unpermute, SM grad
 * reduce-scatter); out[19] whole step; out[20] restore start offset; out[21]
 * restore issue-to-join time; out[22] forward top -> first phase (layout
 * snapshot + H2D); out[23] idle gap between the previous step's end and this
 * step's top; out[24] host time blocked on the planner per step; out[25] / out[26]
 * forward top -> histogram on the host / -> planner callback done; out[27] restore
 * begin -> last copy-engine restore push landed.  n >= 23. */
mp_status mp_fsep_layer_phase_ms(mp_fsep_layer* layer, double* out, uint32_t n);

/* Device-detected failures.  Kernels record them in host-mapped words:
 *   bit 0  receive-buffer overflow (a segment exceeded max_recv_rows; dropped),
 *   bit 1  peer barrier timeout (a rank did not arrive within FSEP_SPIN_TIMEOUT_MS,
 *          default 10 s),
 *   bit 2  restore readiness timeout (a restored expert chunk's flag never
 *          arrived; the gate-up GEMM stopped waiting),
 *   bit 3  memory guard overwritten (checked by mp_fsep_layer_check only: every
 *          internal buffer is followed by a 256-byte guard pattern, verified on
 *          the device -- a kernel wrote past the end of a buffer).
 * Every mp_fsep_layer_forward / _backward / _graph_step / _stats call first
 * reports the words that have landed (MP_ERR_DEVICE, message naming the causes,
 * words cleared).  mp_fsep_layer_check synchronises the device first, so it sees
 * every step enqueued so far; *bits (may be NULL) gets the set bits.  Like every
 * error of this ABI (capi.cpp:54-70), the failure is returned, never thrown. */
mp_status mp_fsep_layer_check(mp_fsep_layer* layer, uint32_t* bits);
/* Test hook forcing a failure condition: "drop_restore_flag" (copy-engine mode:
 * the next restore skips one readiness flag -> bit 2), "barrier_timeout"
 * (virtual mode: emulated rank 0 enters a peer barrier alone -> bit 1),
 * "overwrite_guard" (one byte past the first buffer -> bit 3); "clear_errors" drops
 * the error words that have landed without reporting them (profiling probes only). */
mp_status mp_fsep_layer_debug_inject(mp_fsep_layer* layer, const char* what);
/* Transport probe: `iters` back-to-back full shard restores of the current layout
 * through the push transport (copy engines, or the SM push kernel with
 * FSEP_COMM=sm), each closed by a cross-rank barrier; *ms = mean time per restore. */
mp_status mp_fsep_layer_debug_restore(mp_fsep_layer* layer, int iters, double* ms);

/* Capture forward+backward into a CUDA graph and replay it (bench path). */
mp_status mp_fsep_layer_graph_step(mp_fsep_layer* layer, const void* x, const float* bias, uint32_t n_tokens,
                                   void* y, const void* dy, void* dx, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MOEPLAN_FSEP_H_ */
