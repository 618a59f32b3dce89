"""FSEP MoE-layer step benchmark (forward + backward) on B200.

  python bench.py [--gpus N --steps K --warmup W] [--config mixtral|fine|tiny]
                  [--impl ours|reference] [--alpha 1.2] [--layout laer|static]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step = one forward + backward of the FSEP MoE layer over one batch of
synthetic tokens per GPU (Gumbel-top-k routing with Zipf(alpha) popularity).
`value` is whole-job tokens/s with inputs resident in HBM (device time, max over
ranks); `e2e` is the same step through the public API with the step's inputs
copied from pinned host memory and a result metric read back, inside the timed
region.  Rank 0 prints one JSON line.

--impl reference times the reference's CPU path on the host cores: the
reference planner itself (oracle/_ref: plan_layout + lite_routing, 1 core) plus
the CPU layer restatement (oracle/layer_oracle.py, numpy fp32 on all cores) on a
bounded token sample -- the reference ships no GPU executor.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FSEP MoE-layer fwd+bwd tokens/s at 1/2/4/8 B200, skewed routing; % roofline"
CONFIGS = {
    "mixtral": dict(E=8, K=2, H=4096, F=14336, T=16384,
                    workload="Mixtral-8x7B MoE layer shape: 8 experts top-2, hidden 4096, ffn 14336, 16K tokens/GPU, bf16"),
    "fine": dict(E=64, K=8, H=2048, F=1408, T=32768,
                 workload="fine-grained MoE: 64 experts top-8, hidden 2048, ffn 1408, 32K tokens/GPU"),
    "multilayer": dict(E=8, K=2, H=4096, F=14336, T=16384, layers=4, drift=(0.3, 0.15),
                       workload="multi-layer dynamic skew: 4 stacked Mixtral-shape layers with drifting "
                                "per-iteration routing, planner re-layout every step"),
    # configs[0]: 4096 tokens over 8 simulated devices -> on one GPU as 8 emulated ranks running the
    # shipped multi-GPU transport (MP_FSEP_FLAG_COPY_ENGINE), C=2, planner re-layout every step
    "tiny": dict(E=8, K=2, H=256, F=512, T=512, virtual_ranks=8, capacity=2,
                 workload="tiny FSEP MoE layer: 8 experts top-2, hidden 256, ffn 512, 4096 tokens over 8 simulated "
                          "devices (8 emulated ranks on one GPU), Zipf(1.2)"),
}
SEED_DATA, SEED_PLANNER = 42, 7


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def default_capacity(E, K, N):
    return E if N == 1 else max(K, min(E, 2 * E // N))


def zipf_bias(rng, T, E, alpha, perm):
    ranks = np.arange(1, E + 1, dtype=np.float64)
    p = ranks ** (-alpha)
    p /= p.sum()
    return (np.log(p[perm])[None, :] + rng.gumbel(size=(T, E))).astype(np.float32)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (the
    profiling recipe's clocks line, every 50 ms; idle-only samples dropped).  One
    nvidia-smi process for all of the job's GPUs, started by local rank 0 only (one
    poller per rank added host-side jitter at N=4); devices=None: no sampling."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        self.devices = devices
        self.proc = None

    def __enter__(self):
        if self.devices is None:
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", ",".join(str(d) for d in self.devices)],
                                         stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start (idle-only samples are dropped)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.result = {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if self.proc is None:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                active = int(r[3].strip(), 16) if len(r) > 3 else 0
                if active == 0x1:  # GPU idle only: a sample outside the kernels (e.g. before the region)
                    continue
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].strip().lower() == "active":
                    reasons.add(n)
        self.result = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                       "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU paths
class CpuReference:
    """The reference CPU path of one layer step, timed on the host cores.

    The reference ships no GPU executor: its CPU path for a layer step
    is the reference planner itself (oracle/_ref = the unmodified reference library:
    plan_layout + lite_routing on the step's histogram, 1 core, timed by the
    reference-linked oracle/refplan_bench) plus the CPU restatement of the layer
    math (oracle/layer_oracle.py, numpy fp32, BLAS on all cores).  A step processes
    `sample` tokens in full (all tokens of the workload for the tiny config, a
    bounded sample of the same workload otherwise) and is measured, not modelled:
    tokens/s = sample / (layer-math seconds + planner seconds)."""

    def __init__(self, cfg, N, C, alpha, sample):
        from oracle import layer_oracle as LO
        from oracle import ref as REF
        self.LO, self.REF = LO, REF
        E, K, H, F = cfg["E"], cfg["K"], cfg["H"], cfg["F"]
        self.N, self.C, self.K, self.H, self.F, self.E = N, C, K, H, F, E
        rng = np.random.default_rng(SEED_DATA)
        bf = LO.bf16_round
        nrm = lambda *shape: rng.standard_normal(size=shape, dtype=np.float32)
        self.wg = bf(nrm(E, H) * 0.02)
        self.w1 = np.stack([bf(nrm(F, H) / np.float32(np.sqrt(H))) for _ in range(E)])
        self.w3 = np.stack([bf(nrm(F, H) / np.float32(np.sqrt(H))) for _ in range(E)])
        self.w2 = np.stack([bf(nrm(H, F) / np.float32(np.sqrt(F))) for _ in range(E)])
        perm = rng.permutation(E)
        ranks = N if sample >= N * cfg["T"] else 1  # full tiny step: every simulated rank's tokens
        per = sample // ranks
        self.xs = [bf(nrm(per, H)) for _ in range(ranks)]
        self.dys = [bf(nrm(per, H) * 0.1) for _ in range(ranks)]
        self.bias = [zipf_bias(rng, per, E, alpha, perm) for _ in range(ranks)]
        self.sample = per * ranks
        self.full = ranks == N and N > 1
        # the planner's input: the histogram of the full-size step (every rank's T tokens)
        scale = cfg["T"] // 4096 if cfg["T"] >= 4096 else 1
        tk = min(cfg["T"], 4096)
        self.R = np.stack([np.bincount(LO.topk(zipf_bias(rng, tk, E, alpha, perm), K)[0].reshape(-1), minlength=E)
                           for _ in range(N)]) * scale
        self.planner = N > 1 and REF.available()
        self.A = None
        if self.full:
            from paper_2602_11686_b200 import planner as PL
            self.A = PL.even_replication_layout(N, E, C)

    def step(self):
        """One measured step; returns (seconds, tokens, planner seconds)."""
        plan_s = 0.0
        if self.planner:
            res = self.REF.plan_bench(self.R.tolist(), self.C, 20, bandwidth=9e11, v_comm=2.0 * self.H,
                                      v_comp=6.0 * self.H * self.F, b_comp=1.6354e15)
            plan_s = (res["plan_us"] + res["route_us"]) * 1e-6
        t0 = time.perf_counter()
        self.LO.layer_step(self.xs, self.bias, self.wg, self.w1, self.w3, self.w2, self.K, self.A, self.C, self.dys,
                           dtype=np.float32)
        layer_s = time.perf_counter() - t0
        return layer_s + plan_s, self.sample, plan_s

    def describe(self, cfg_name):
        planner = ("reference plan_layout + lite_routing (oracle/_ref, 1 core) on the step's N x E histogram"
                   if self.planner else "no planner call (N=1: one device hosts every expert)")
        what = (f"all {self.sample} tokens of the {cfg_name} step ({self.N} simulated ranks, routed through "
                f"lite_routing into the planned layout)" if self.full else
                f"{self.sample} tokens of the {cfg_name} workload per step")
        return (f"{what}: layer math via oracle/layer_oracle.py (numpy fp32 BLAS, all host cores) + "
                f"{planner}; measured per step, tokens/s = tokens / step seconds")


def cpu_sample_tokens(cfg, N, budget_flops):
    if cfg.get("virtual_ranks"):
        return cfg["virtual_ranks"] * cfg["T"]  # the tiny step in full
    return max(64, min(2048, int(budget_flops / (18 * cfg["K"] * cfg["H"] * cfg["F"]))))


def use_all_host_cores():
    """torchrun sets OMP_NUM_THREADS=1 for every rank; the CPU reference path runs on rank 0
    alone and should use every host core, so lift the BLAS thread limit at run time.
    Returns the BLAS thread count in effect."""
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        threadpool_limits(limits=os.cpu_count(), user_api="blas")
        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))


def run_reference_impl(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = use_all_host_cores()
    N = cfg.get("virtual_ranks") or args.gpus
    C = args.capacity or cfg.get("capacity") or default_capacity(cfg["E"], cfg["K"], N)
    sample = args.cpu_sample or cpu_sample_tokens(cfg, N, 2.0e12)
    ref = CpuReference(cfg, N, C, args.alpha, sample)
    ts, toks, plan = [], 0, 0.0
    for i in range(args.warmup + args.steps):
        sec, n, ps = ref.step()
        if i >= args.warmup:
            ts.append(sec)
            toks += n
            plan += ps
    rate = toks / sum(ts)
    cpu = {"value": rate, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": ref.describe(args.config),
           "planner_us_per_step": round(plan / len(ts) * 1e6, 2)}
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(ts) / len(ts) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Gumbel-top-k Zipf routing, random-init weights)",
            "config": {"workload": cfg["workload"], "n_experts": cfg["E"], "top_k": cfg["K"], "hidden": cfg["H"],
                       "ffn": cfg["F"], "tokens_per_gpu": cfg["T"], "capacity": C, "zipf_alpha": args.alpha,
                       "tokens_per_step_measured": ref.sample},
            "cpu_baseline": cpu,
            "e2e": {"value": rate, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU path
def token_kernel_bandwidth(phases, layer, PL, N, rank, T, K, H, F=0, C=0, config=None):
    """HBM and NVLink throughput of the token-movement kernels (rank 0's layer 0).

    Algorithmic bytes per step (bf16 rows of H elements, T tokens, K slots each):
      dispatch    read x (T*H*2)              + write T*K rows into the owners' arenas
      combine     read T*K rows (local/peer)   + write y (T*H*2)
      unpermute   read T*K dx rows (local/peer) + write dx (T*H*2)
    The remote share (rows whose slot lives on another GPU, i.e. NVLink traffic)
    comes from lite_routing(R, A) of the step's histogram and layout.
    With F and C (N > 1): the shard restore, C hosted experts x (N-1)/N of their
    3*H*F bf16 parameters received over NVLink per step (copy-engine pushes), over
    the time from the restore's start to its last push landing (phase
    restore_landed_ms; else the issue-to-join interval, a lower bound on the rate).
    """
    row = H * 2
    remote = 0
    if N > 1:
        R = layer.histogram()
        A = layer.read("layout").reshape(R.shape[1], N)
        S = PL.lite_routing(R, A)[rank]  # [E, dst]
        if getattr(layer.spec, "local_first", False):
            for e in range(S.shape[0]):
                if A[e, rank]:
                    S[e, :] = 0
                    S[e, rank] = R[rank, e]
        remote = int(S.sum() - S[:, rank].sum())
    out = {}
    for name, ph in (("dispatch", "dispatch"), ("combine", "combine"), ("unpermute", "unpermute")):
        ms = phases.get(ph) or 0.0
        if ms <= 0:
            continue
        b = T * row + T * K * row
        out[name] = {"ms": round(ms, 4), "bytes": b, "GBps": round(b / (ms * 1e-3) / 1e9, 1),
                     "remote_rows": remote, "nvlink_GBps": round(remote * row / (ms * 1e-3) / 1e9, 1)}
    hbm = peaks()[2]
    for v in out.values():
        v["hbm_frac"] = round(v["GBps"] / hbm, 4)
    # the same kernels timed alone (committed ncu launch list of this config at N=1): in the
    # step they run at the power-capped SM clock right after the GEMMs
    if N == 1 and config:
        launches = ROOT / "profiles" / "r02" / f"launches_n1_{config}_final3.txt"
        kern = {"dispatch": "dispatch_tma_kernel", "combine": "combine_kernel<", "unpermute": "unpermute_bwd_kernel"}
        if launches.exists():
            for line in launches.read_text().splitlines():
                parts = [p_.strip() for p_ in line.split("|")]
                for name, key in kern.items():
                    if name in out and len(parts) == 5 and key in parts[0] and not line.startswith("#"):
                        iso = float(parts[3])
                        out[name]["isolated_ms"] = iso
                        out[name]["isolated_hbm_frac"] = round(out[name]["bytes"] / (iso * 1e-3) / 1e9 / hbm, 4)
                        out[name]["isolated_source"] = str(launches.relative_to(ROOT))
    rms = phases.get("restore_landed_ms") or phases.get("restore_ms") or 0.0
    if N > 1 and F and C and rms > 0:
        b = C * 3 * H * F * 2 * (N - 1) // N
        out["restore"] = {"ms": round(rms, 4), "bytes": b, "effective_GBps_per_sending_gpu": round(b / (rms * 1e-3) / 1e9, 1),
                          "note": "effective restore throughput of this (sending) GPU: its copy-engine pushes from the "
                                  "restore's start to its last push landing (slots >= 1 are held back until dispatch "
                                  "ends, so this is a lower bound on the link rate; raw rates: tools/transport_probe.py)"
                                  if phases.get("restore_landed_ms") else
                                  "copy-engine pushes under the forward; issue-to-join interval"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral", choices=list(CONFIGS))
    ap.add_argument("--alpha", type=float, default=1.2)
    ap.add_argument("--layout", default="laer", choices=["laer", "static"])
    ap.add_argument("--capacity", type=int, default=0)
    ap.add_argument("--tokens", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-static", action="store_true")
    ap.add_argument("--no-ep", action="store_true", help="skip the pure expert-parallel comparison (N>1)")
    ap.add_argument("--routing", default="lite", choices=["lite", "local_first"],
                    help="token routing: the reference lite_routing (default) or the local-first variant")
    ap.add_argument("--no-local-first", action="store_true", help="skip the local-first routing comparison (N>1)")
    ap.add_argument("--no-prefetch", action="store_true",
                    help="multi-layer: do not chain layers (each layer restores at its own forward)")
    ap.add_argument("--no-phases", action="store_true", help="skip per-phase device timing events")
    ap.add_argument("--defer-rs", action="store_true",
                    help="multi-layer: complete each layer's gradient reduce-scatter under the previous layer's "
                         "backward (PAPER Fig.5(e))")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.tokens:
        cfg["T"] = args.tokens
    if args.warmup < 3:
        args.warmup = 3  # contract: at least 3 untimed warm-up steps
    if args.impl == "reference":
        return run_reference_impl(args, cfg)

    if not args.no_phases:
        os.environ.setdefault("FSEP_PHASE_TIMING", "1")
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # V > 0: the configuration's N ranks are emulated on this one GPU (tiny config)
    V = cfg.get("virtual_ranks", 0) if world == 1 else 0
    N = V or world
    E, K, H, F, T = cfg["E"], cfg["K"], cfg["H"], cfg["F"], cfg["T"]
    C = args.capacity or cfg.get("capacity") or default_capacity(E, K, N)
    L = cfg.get("layers", 1)
    RT = (V or 1) * T  # token rows this process feeds per step

    from paper_2602_11686_b200 import planner as PL
    from paper_2602_11686_b200.layer import FsepLayer, LayerSpec

    cfg_json = json.dumps({"topology": {"n_nodes": 1, "devices_per_node": N, "b_intra": 9e11, "b_inter": 9e11},
                           "cost": {"v_comm": 2.0 * H, "v_comp": 6.0 * H * F, "b_comp": peaks()[0] * 1e12},
                           "model": {"n_experts": E, "capacity": C}, "planner": {"seed": SEED_PLANNER}})
    def make_layers(cap, layout, resident=False, local_first=False):
        out = []
        for l in range(L):
            layer = FsepLayer(LayerSpec(E, K, H, F, T, cap, world=N, rank=rank, virtual=V > 0, resident=resident,
                                        local_first=local_first, copy_engine=V > 0, defer_rs=args.defer_rs))
            if world > 1:
                layer.connect_torch_distributed()
            # random-init weights of the named architecture (identical on every rank)
            g = torch.Generator(device="cuda").manual_seed(SEED_DATA + 7919 * l)
            for e in range(E):
                w1 = (torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16()
                w3 = (torch.randn(F, H, device="cuda", generator=g) / H ** 0.5).bfloat16()
                w2 = (torch.randn(H, F, device="cuda", generator=g) / F ** 0.5).bfloat16()
                layer.load_expert(e, w1, w3, w2)
            layer.load_router((torch.randn(E, H, device="cuda", generator=g) * 0.02).bfloat16())
            if N > 1 and layout == "laer":
                layer.attach_planner(PL.Config(cfg_json), layer=l)
            elif N > 1:
                layer.set_layout(PL.static_ep_layout(N, E, cap))
            out.append(layer)
        if L > 1 and N > 1 and not args.no_prefetch:  # Fig.5: layer l+1's restore under layer l's MLP
            for l in range(L - 1):
                out[l].chain(out[l + 1])
        torch.cuda.synchronize()
        return out

    layers = make_layers(C, args.layout, local_first=args.routing == "local_first")
    # synthetic data: x ~ N(0,1), dy ~ N(0, 0.1^2), per-rank seeds; routing bias generated on the host:
    # Gumbel-top-k with Zipf(alpha) popularity, or (multi-layer config) the drifting per-iteration
    # popularity of the reference trace generator (generate_trace: Dirichlet(0.3) init, sigma 0.15 walk).
    gx = torch.Generator(device="cuda").manual_seed(SEED_DATA * 1000 + rank)
    x = torch.randn(RT, H, device="cuda", generator=gx).bfloat16()
    dy = (torch.randn(RT, H, device="cuda", generator=gx) * 0.1).bfloat16()
    rng = np.random.default_rng(SEED_DATA + rank)
    n_bias = args.warmup + args.steps if cfg.get("drift") else 4
    if cfg.get("drift"):
        spec = json.dumps({"n_devices": N, "n_experts": E, "n_layers": L, "n_iterations": n_bias,
                           "tokens_per_device": T, "skew_alpha": cfg["drift"][0], "drift_sigma": cfg["drift"][1],
                           "seed": SEED_DATA})
        logp = np.log(np.maximum(PL.trace_popularity(spec), 1e-30))
        gum = [rng.gumbel(size=(RT, E)) for _ in range(4)]
        bias_h = [[torch.from_numpy((logp[l, i][None, :] + gum[(i + l) % 4]).astype(np.float32)).pin_memory()
                   for i in range(n_bias)] for l in range(L)]
    else:
        perm = np.random.default_rng(SEED_DATA).permutation(E)  # same popularity order on all ranks
        bias_h = [[torch.from_numpy(zipf_bias(rng, RT, E, args.alpha, perm)).pin_memory() for _ in range(n_bias)]
                  for _ in range(L)]
    bias_d = [[b.cuda() for b in row] for row in bias_h]
    ys = [torch.empty_like(x) for _ in range(L)]
    dxs = [torch.empty_like(x) for _ in range(L)]
    stream = torch.cuda.current_stream()

    def run_step(i, xin, dyin, biases, y_last=None, dx_first=None):
        h = xin
        for l, layer in enumerate(layers):
            out = y_last if (l == L - 1 and y_last is not None) else ys[l]
            layer.forward(h, biases[l][i % n_bias], T, out)
            h = out
        gr = dyin
        for l in reversed(range(L)):
            out = dx_first if (l == 0 and dx_first is not None) else dxs[l]
            layers[l].backward(gr, out)
            gr = out

    def assert_healthy(tag):
        # a step with a device-detected failure (receive overflow, barrier or readiness
        # timeout) must not produce a bench line: MP_ERR_DEVICE raises here, on every rank
        for l, layer in enumerate(layers):
            try:
                layer.check()
            except Exception as exc:
                raise SystemExit(f"bench: {tag}: layer {l} on rank {rank} failed on the device: {exc}")

    def step(i):
        run_step(i, x, dy, bias_d)

    # L2 rule: a workload whose per-step bytes (x, dy, y, dx, every expert's weights) exceed
    # twice the L2 runs back to back; a smaller one (the tiny configs[0] step) gets the L2
    # flushed by a 2x-L2 write before every timed step, outside that step's events
    l2_bytes = int(getattr(torch.cuda.get_device_properties(0), "L2_cache_size", 126 << 20))
    step_bytes = 4 * x.numel() * 2 + L * E * 3 * H * F * 2
    flush_l2 = step_bytes < 2 * l2_bytes
    flush_buf = torch.empty(2 * l2_bytes, dtype=torch.uint8, device="cuda") if flush_l2 else None
    l2_note = (f"L2 flushed before every timed step ({2 * l2_bytes >> 20} MiB write, outside the step's events; "
               f"per-step bytes {step_bytes >> 20} MiB < 2x L2)" if flush_l2 else
               f"inputs larger than L2 (per-step bytes {step_bytes >> 20} MiB: x {x.numel() * 2 >> 20} MiB + weights)")

    def timed(nsteps, fn, flush=None):
        flush = flush_l2 if flush is None else flush
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if flush:
            evs = []
            for i in range(nsteps):
                flush_buf.fill_(i & 0xFF)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                fn(i)
                e.record(stream)
                evs.append((s, e))
            torch.cuda.synchronize()
            ms = sum(s.elapsed_time(e) for s, e in evs) / nsteps
        else:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            for i in range(nsteps):
                fn(i)
            e.record(stream)
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / nsteps
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    # the clock sampler runs from before the warm-up steps to the end of the timed
    # region, so it sees the GPU under load through the whole measured window
    nloc = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    with ClockSampler(list(range(nloc)) if local == 0 else None) as clk:
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        for layer in layers:
            layer.stats_reset()
        ms = timed(args.steps, lambda i: step(args.warmup + i))
    clocks = clk.result
    assert_healthy("timed steps")
    sts = [layer.stats() for layer in layers]
    phases = layers[0].phase_ms() if os.environ.get("FSEP_PHASE_TIMING") == "1" else None
    if phases:
        phases["fwd_gemms"] = round(phases["fwd_gemm_gateup"] + phases["fwd_gemm_down"], 4)
    comm = token_kernel_bandwidth(phases, layers[0], PL, N, rank, T, K, H, F, C, config=args.config) if phases else None
    per_rank = None
    if world > 1 and phases:
        # per-rank view of the phases that expose load imbalance (barrier waits absorb it)
        allp = [None] * world
        rows = int(layers[0].read("total_rows").view(np.int32)[0])
        dist.all_gather_object(allp, {"phases": phases, "gemm_ms": sum(s_["gemm_ms"] for s_ in sts), "rows": rows})
        keys = ["router_scan", "dispatch", "fwd_gemm_gateup", "fwd_gemm_down", "fwd_gemms", "fwd_barrier", "combine_bwd_router_wgrad", "bwd_gemms",
                "rs_push_wait", "rs_barrier", "rs_sum", "step_total"]
        per_rank = {k: [round(a["phases"].get(k, 0.0), 3) for a in allp] for k in keys}
        per_rank["gemm_ms"] = [round(a["gemm_ms"], 3) for a in allp]
        per_rank["recv_rows_last_step"] = [a["rows"] for a in allp]
    st = {"gemm_ms": sum(s_["gemm_ms"] for s_ in sts), "gemm_flops": sum(s_["gemm_flops"] for s_ in sts),
          "kernel_launches": sum(s_["kernel_launches"] for s_ in sts)}
    value = N * T / (ms * 1e-3)  # whole job: every rank's (or emulated rank's) T tokens

    # ---- roofline of the dominant kernel class (grouped tcgen05 GEMMs)
    burst, sustained, hbm, src = peaks()
    gemm_tflops = st["gemm_flops"] / (st["gemm_ms"] * 1e-3) / 1e12
    flop_tok = 18.0 * K * H * F * L
    n_dev = world  # physical GPUs the step ran on
    traffic = pipe_pct = prof_src = None
    prof = ROOT / "profiles" / f"gemm_traffic_{args.config}.json"
    if prof.exists():  # from the committed ncu --set full capture of this config (tools/ncu_summary.py)
        try:
            pj = json.loads(prof.read_text())
            traffic, pipe_pct, prof_src = pj.get("dram_bytes_per_launch"), pj.get("tensor_pipe_active_pct"), pj.get("source")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": round(gemm_tflops, 1), "peak": sustained, "unit": "TFLOP/s",
                "frac": round(gemm_tflops / sustained, 4), "traffic": traffic,
                "kernel": f"grouped tcgen05 GEMMs ({6 * L} launches/step: gate-up+SwiGLU, down, 2 dgrad, 2 wgrad"
                          f"{' per layer' if L > 1 else ''})",
                "flops_per_step": st["gemm_flops"], "gemm_ms_per_step": round(st["gemm_ms"], 4),
                "peak_source": f"MEASURED_PEAKS.json bf16_tflops_sustained ({src}); burst {burst}",
                "frac_of_burst": round(gemm_tflops / burst, 4),
                "tensor_pipe_active_pct": pipe_pct, "ncu_source": prof_src,
                "step_frac": round(value / n_dev * flop_tok / (sustained * 1e12), 4)}

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # Public-API step with host inputs: every step's x, dy and routing biases are
        # copied H2D from pinned memory (double-buffered on a copy stream, so step
        # i+1's upload overlaps step i's compute) and a result metric is read back.
        x_h = x.cpu().pin_memory()
        dy_h = dy.cpu().pin_memory()
        bufs = [(torch.empty_like(x), torch.empty_like(dy), [torch.empty_like(bias_d[0][0]) for _ in range(L)])
                for _ in range(2)]
        # the step's outputs (last layer's y, first layer's dx) come back to pinned host memory
        # every step on a D2H stream, double-buffered so step i's copy overlaps step i+1
        outs = [(torch.empty_like(x), torch.empty_like(x)) for _ in range(2)]
        outs_h = [(torch.empty(x.shape, dtype=x.dtype).pin_memory(), torch.empty(x.shape, dtype=x.dtype).pin_memory())
                  for _ in range(2)]
        copy_stream = torch.cuda.Stream()
        d2h_stream = torch.cuda.Stream()
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]
        for ev in free + drained:
            ev.record(stream)

        def upload(i):
            b = i % 2
            copy_stream.wait_event(free[b])
            with torch.cuda.stream(copy_stream):
                bufs[b][0].copy_(x_h, non_blocking=True)
                bufs[b][1].copy_(dy_h, non_blocking=True)
                for l in range(L):
                    bufs[b][2][l].copy_(bias_h[l][i % n_bias], non_blocking=True)
            ready[b].record(copy_stream)

        metric_h = [torch.empty(2, dtype=torch.float32).pin_memory() for _ in range(2)]
        full_outputs = [True]

        def e2e_step(i):
            b = i % 2
            if i == 0:
                upload(0)
            # next step's inputs are queued before this step's work (they wait only for the
            # step that last used their buffer), so the H2D copies are not stuck behind
            # this step's copy-engine restore / reduce-scatter pushes
            upload(i + 1)
            stream.wait_event(ready[b])
            stream.wait_event(drained[b])  # step i-2's outputs have left this buffer
            xb, dyb, bb = bufs[b]
            run_step(0, xb, dyb, [[t] for t in bb], y_last=outs[b][0], dx_first=outs[b][1])
            free[b].record(stream)
            computed[b].record(stream)
            d2h_stream.wait_event(computed[b])
            with torch.cuda.stream(d2h_stream):
                if full_outputs[0]:
                    outs_h[b][0].copy_(outs[b][0], non_blocking=True)
                    outs_h[b][1].copy_(outs[b][1], non_blocking=True)
                else:  # the step's result metric only: [sum y, sum dx]
                    m = torch.stack([outs[b][0].sum(dtype=torch.float32), outs[b][1].sum(dtype=torch.float32)])
                    metric_h[b].copy_(m, non_blocking=True)
            drained[b].record(d2h_stream)

        bi = x.numel() * 2 + dy.numel() * 2 + L * bias_d[0][0].numel() * 4
        runs = {}
        for full in (False, True):
            full_outputs[0] = full
            for i in range(args.warmup):
                e2e_step(i)
            torch.cuda.synchronize()
            # continuous timing (no L2 flush): the step's inputs arrive fresh from the host
            # every step, and the H2D / D2H copies overlap neighbouring steps
            runs[full] = timed(args.steps, e2e_step, flush=False)  # its closing synchronize waits for the last D2H
            assert_healthy("e2e steps")
        ems = runs[False]
        e2e = {"value": N * T / (ems * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": 8,
               "ms_per_step": ems,
               "note": "public-API step: x, dy, routing bias H2D from pinned host memory every step (double-buffered "
                       "copy stream) and the step's result metric [sum y, sum dx] D2H every step, inside the timed "
                       "region (y and dx feed the neighbouring layers on the device inside a model)",
               "with_outputs_d2h": {"value": N * T / (runs[True] * 1e-3), "ms_per_step": runs[True],
                                    "d2h_bytes_per_step": 2 * x.numel() * 2,
                                    "note": "same, plus the full outputs y (last layer) and dx (first layer) "
                                            "copied D2H into pinned host memory every step (double-buffered)"}}

    # ---- static-EP comparison (same kernels, static_ep_layout at the same C)
    static = None
    if N > 1 and not V and args.layout == "laer" and not args.no_static:
        for layer in layers:
            layer.detach_planner()
            layer.set_layout(PL.static_ep_layout(N, E, C))
        for i in range(args.warmup):
            step(i)
        sms = timed(args.steps, lambda i: step(args.warmup + i))
        assert_healthy("static-EP steps")
        static = {"value": N * T / (sms * 1e-3), "ms_per_step": sms, "layout": "static_ep_layout(N,E,C)",
                  "speedup_laer_over_static": round(sms / ms, 4)}

    # ---- pure expert parallelism: C = E/N, one host per expert, experts
    # resident across steps, no restore and no gradient reduce-scatter -- same kernels
    pure_ep = None
    if N > 1 and not V and args.layout == "laer" and not args.no_ep and E % N == 0:
        for layer in layers:
            layer.close()
        torch.cuda.empty_cache()
        layers = make_layers(E // N, "static", resident=True)
        for i in range(args.warmup):
            step(i)
        ems_ = timed(args.steps, lambda i: step(args.warmup + i))
        assert_healthy("pure-EP steps")
        pure_ep = {"value": N * T / (ems_ * 1e-3), "ms_per_step": ems_, "capacity": E // N,
                   "layout": "static_ep_layout(N,E,E/N), experts resident, no restore / reduce-scatter",
                   "speedup_laer_over_ep": round(ems_ / ms, 4)}

    # ---- local-first token routing (NOT the reference lite_routing)
    local_first = None
    if N > 1 and not V and args.layout == "laer" and args.routing == "lite" and not args.no_local_first:
        for layer in layers:
            layer.close()
        torch.cuda.empty_cache()
        layers = make_layers(C, "laer", local_first=True)
        for i in range(args.warmup):
            step(i)
        lms = timed(args.steps, lambda i: step(args.warmup + i))
        assert_healthy("local-first steps")
        local_first = {"value": N * T / (lms * 1e-3), "ms_per_step": lms,
                       "routing": "local-first (non-parity variant): sources hosting a replica keep their tokens",
                       "speedup_over_lite_routing": round(ms / lms, 4)}

    # ---- CPU baseline (rank 0 at N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = use_all_host_cores()
        ref = CpuReference(cfg, N, C, args.alpha, args.cpu_sample or cpu_sample_tokens(cfg, N, 2.0e12))
        sec, ntok, ps = ref.step()
        cpu = {"value": ntok / sec, "unit": "tokens/s", "cores": threads, "kind": "port",
               "sample": ref.describe(args.config), "seconds": round(sec, 3),
               "planner_us_per_step": round(ps * 1e6, 2)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic: x~N(0,1) bf16, random-init weights, Gumbel-top-k routing with Zipf popularity",
                "config": {"workload": cfg["workload"], "n_experts": E, "top_k": K, "hidden": H, "ffn": F,
                           "tokens_per_gpu": T, "capacity": C, "layers": L,
                           "routing": ("drifting trace popularity alpha=%g sigma=%g" % tuple(cfg["drift"]))
                           if cfg.get("drift") else f"Zipf({args.alpha}) Gumbel-top-k",
                           "layout": args.layout if N > 1 else "single device (C=E)",
                           "emulated_ranks": V or None,
                           "token_routing": "lite_routing (reference, planner.cpp:238-287)" if args.routing == "lite"
                           else "local-first (non-parity variant)",
                           "parallelism": f"fsep{N}" + (" (emulated on 1 GPU)" if V else ""),
                           "defer_rs": bool(args.defer_rs),
                           "cross_layer_prefetch": L > 1 and N > 1 and not args.no_prefetch, "l2": l2_note},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": st["kernel_launches"] *
                args.steps, "clocks": clocks}
        if static:
            line["static_ep"] = static
        if pure_ep:
            line["pure_ep"] = pure_ep
        if local_first:
            line["local_first_routing"] = local_first
        if phases:
            line["phases_ms_layer0"] = phases
        if comm:
            line["token_kernels_layer0"] = comm
        if per_rank:
            line["phases_ms_per_rank_layer0"] = per_rank
        print(json.dumps(line), flush=True)
    for layer in layers:
        layer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
