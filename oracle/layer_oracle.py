"""ORACLE (test infrastructure only): numpy restatement of the FSEP MoE-layer step.

Parity status: the reference (/root/reference/proj) contains no router, FFN,
dispatch or combine numerics (its GPU executor is out of its scope,
/root/reference/SPEC.md:8), so this oracle is written from the paper and is
"parity unpinned" for the floating-point parts:
  * gating      g(x) = Softmax(TopK(x W_g^T))
  * expert FFN  SwiGLU, 6*H*F forward FLOPs per token
  * FSEP shard / unshard / reshard semantics
The COUNT-level parts are pinned to the reference: the routing matrix R, the
layout A (planner), lite routing S (planner.cpp:238-287) -- via
oracle/planner_port.py, itself pinned against the reference library.

Bit-exact parts (must match the GPU exactly):
  * router logits in the canonical order the kernel uses (one sequential fp32
    accumulation over h, then + bias) -- products of two bf16 values are exact
    in fp32, so FMA on the GPU equals multiply-then-add here;
  * top-k (largest logit, lowest expert id on ties), R, S, every token-slot's
    destination (device, row) and the per-device segment layout.
Floating-point parts (outputs, gradients) are computed in fp32 (float64 for the
reductions) from the same bf16-representable inputs; the tolerance lives in the
tests.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

from . import planner_port as P


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    u = np.array(a, dtype=np.float32, copy=True).view(np.uint32)
    u += np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    u &= np.uint32(0xFFFF0000)
    return u.view(np.float32)


# ------------------------------------------------------------------- router
def router_logits(x: np.ndarray, wg: np.ndarray, bias: np.ndarray | None) -> np.ndarray:
    """Canonical-order fp32 logits [T, E]: one sequential fp32 accumulation over
    h (products of bf16 values are exact in fp32, so this equals the kernel's
    FMA chain in csrc/kernels/router.cu), then + bias."""
    T, H = x.shape
    xv = np.ascontiguousarray(x.astype(np.float32).T)    # [H, T]
    wv = np.ascontiguousarray(wg.astype(np.float32).T)   # [H, E]
    acc = np.zeros((T, wg.shape[0]), dtype=np.float32)
    for h in range(H):
        acc += xv[h][:, None] * wv[h][None, :]
    if bias is not None:
        acc = acc + bias.astype(np.float32)
    return acc


def topk(logits: np.ndarray, k: int):
    """Top-k ids (ties -> lowest id) and softmax-over-selected weights."""
    idx = np.argsort(-logits, axis=1, kind="stable")[:, :k].astype(np.int32)
    sel = np.take_along_axis(logits, idx, axis=1).astype(np.float64)
    w = np.exp(sel - sel[:, :1])
    w = w / w.sum(axis=1, keepdims=True)
    return idx, w.astype(np.float32)


# ------------------------------------------------------------------- routing
@dataclass
class Routing:
    idx: List[np.ndarray]        # per rank [T, K]
    w: List[np.ndarray]          # per rank [T, K]
    R: np.ndarray                # [N, E] uint64
    S: np.ndarray                # [N, E, N]
    slot_dev: List[np.ndarray]   # per rank [T, K] destination device
    slot_row: List[np.ndarray]   # per rank [T, K] destination row
    seg_rows: np.ndarray         # [N, C]
    seg_off: np.ndarray          # [N, C]
    slot_expert: np.ndarray      # [N, C]


def route(idx_list, w_list, A: np.ndarray, E: int, C: int, local_first: bool = False) -> Routing:
    """Token-slot destinations under layout A (E x N), following lite routing's
    share/remainder split (planner.cpp:277-282) with slots ranked by token order.

    local_first (NOT the reference algorithm; the runtime's opt-in
    MP_FSEP_FLAG_LOCAL_FIRST variant): a source that hosts a
    replica of e keeps all its e-tokens local; other sources split as above."""
    N = len(idx_list)
    R = np.zeros((N, E), dtype=np.uint64)
    for i, idx in enumerate(idx_list):
        R[i] = np.bincount(idx.reshape(-1), minlength=E)
    topo = P.Topology(1, N, 1.0, 1.0)
    Al = A.astype(int).tolist()
    S = np.zeros((N, E, N), dtype=np.uint64)
    for (s, e, d, tok) in P.lite_routing(R.tolist(), Al, topo):
        S[s, e, d] = tok
    if local_first:
        for s_ in range(N):
            for e in range(E):
                if A[e, s_]:
                    S[s_, e, :] = 0
                    S[s_, e, s_] = R[s_, e]
    hosts = [[d for d in range(N) if A[e, d]] for e in range(E)]
    slot_expert = np.zeros((N, C), dtype=np.int64)
    seg_rows = np.zeros((N, C), dtype=np.int64)
    seg_off = np.zeros((N, C), dtype=np.int64)
    for d in range(N):
        ex = [e for e in range(E) if A[e, d]]
        assert len(ex) == C
        off = 0
        for c, e in enumerate(ex):
            rows = int(S[:, e, d].sum())
            slot_expert[d, c], seg_rows[d, c], seg_off[d, c] = e, rows, off
            off += (rows + 127) // 128 * 128
    slot_dev, slot_row = [], []
    for i, idx in enumerate(idx_list):
        T, K = idx.shape
        dev = np.zeros((T, K), dtype=np.int64)
        row = np.zeros((T, K), dtype=np.int64)
        seen = np.zeros(E, dtype=np.int64)
        for t in range(T):
            for k in range(K):
                e = int(idx[t, k])
                r = seen[e]
                seen[e] += 1
                cum = 0
                for d in hosts[e]:
                    amt = int(S[i, e, d])
                    if r < cum + amt:
                        c = int(np.where(slot_expert[d] == e)[0][0])
                        dev[t, k] = d
                        row[t, k] = seg_off[d, c] + int(S[:i, e, d].sum()) + (r - cum)
                        break
                    cum += amt
        slot_dev.append(dev)
        slot_row.append(row)
    return Routing(list(idx_list), list(w_list), R, S, slot_dev, slot_row, seg_rows, seg_off, slot_expert)


# ------------------------------------------------------------------- numerics
def _silu(g):
    return g / (1.0 + np.exp(-g))


def layer_step(xs, biases, wg, w1, w3, w2, K: int, A: np.ndarray, C: int, dys, dtype=np.float64,
               local_first: bool = False):
    """Forward + backward of the FSEP layer over N ranks.

    xs/dys: per-rank [T, H] (bf16 values as float32); wg [E, H]; w1/w3 [E, F, H];
    w2 [E, H, F].  Returns dict with routing + per-rank y, dx and expert/router grads.
    The numerics are layout-independent (FSEP == FSDP numerically);
    the layout only decides where each token-slot is computed (routing)."""
    N = len(xs)
    E = wg.shape[0]
    idx_l, w_l, logit_l = [], [], []
    for x, b in zip(xs, biases):
        lg = router_logits(x, wg, b)
        idx, w = topk(lg, K)
        idx_l.append(idx)
        w_l.append(w)
        logit_l.append(lg)
    rt = route(idx_l, w_l, A, E, C, local_first) if A is not None else None
    f64 = dtype  # float64 for parity checks; float32 (BLAS sgemm) for the timed CPU baseline
    ys, dxs = [], []
    dW1 = np.zeros(w1.shape, dtype=f64)
    dW3 = np.zeros(w3.shape, dtype=f64)
    dW2 = np.zeros(w2.shape, dtype=f64)
    dWg = []
    for i in range(N):
        x = xs[i].astype(f64, copy=False)
        dy = dys[i].astype(f64, copy=False)
        T, H = x.shape
        idx, w = idx_l[i], w_l[i].astype(f64, copy=False)
        y = np.zeros((T, H), dtype=f64)
        dx = np.zeros((T, H), dtype=f64)
        dw = np.zeros((T, K), dtype=f64)
        for e in range(E):
            tk = np.argwhere(idx == e)
            if len(tk) == 0:
                continue
            t, k = tk[:, 0], tk[:, 1]
            xe = x[t]
            g = xe @ w1[e].astype(f64, copy=False).T
            u = xe @ w3[e].astype(f64, copy=False).T
            sg = 1.0 / (1.0 + np.exp(-g))
            a = g * sg * u
            ye = a @ w2[e].astype(f64, copy=False).T
            y[t] += w[t, k][:, None] * ye
            dw[t, k] = np.sum(dy[t] * ye, axis=1)
            dye = w[t, k][:, None] * dy[t]
            da = dye @ w2[e].astype(f64, copy=False)
            du = da * g * sg
            dg = da * u * sg * (1.0 + g * (1.0 - sg))
            dx[t] += dg @ w1[e].astype(f64, copy=False) + du @ w3[e].astype(f64, copy=False)
            dW2[e] += dye.T @ a
            dW1[e] += dg.T @ xe
            dW3[e] += du.T @ xe
        dl = w * (dw - np.sum(w * dw, axis=1, keepdims=True))
        dWg_i = np.zeros((E, H), dtype=f64)
        for k in range(K):
            dx += dl[:, k:k + 1] * wg.astype(f64, copy=False)[idx[:, k]]
            np.add.at(dWg_i, idx[:, k], dl[:, k:k + 1] * x)
        ys.append(y)
        dxs.append(dx)
        dWg.append(dWg_i)
    return {"routing": rt, "logits": logit_l, "y": ys, "dx": dxs, "dW1": dW1, "dW3": dW3, "dW2": dW2, "dWg": dWg}


def make_bias(rng: np.random.Generator, T: int, E: int, alpha: float, perm=None, scale: float = 1.0) -> np.ndarray:
    """Gumbel-top-k routing bias ln p_j + Gumbel for a Zipf(alpha) popularity over
    a seeded expert permutation; fp32, generated on the host."""
    ranks = np.arange(1, E + 1, dtype=np.float64)
    p = ranks ** (-alpha)
    p /= p.sum()
    if perm is not None:
        p = p[perm]
    g = rng.gumbel(size=(T, E))
    return (scale * (np.log(p)[None, :] + g)).astype(np.float32)
