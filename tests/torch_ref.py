"""Plain torch fp32 reference of the FSEP layer step's floating-point math, on the GPU
(test infrastructure: the oracle's numpy restatement, oracle/layer_oracle.py:layer_step,
is too slow at the bench shapes, so the full-size tests recompute the same math here).

Routing (top-k ids and softmax weights) comes from the numpy oracle
(layer_oracle.router_logits + topk: bit-exact with the GPU router); everything
after it follows layer_oracle.layer_step line by line in fp32 torch matmuls
(TF32 disabled):
  y_t   = sum_k w_tk * W2_e (silu(W1_e x_t) * W3_e x_t)
  dx_t  = sum_k [W1_e^T dg + W3_e^T du]  +  sum_k dl_tk * Wg[e_k]
  dW*_e = sum over every rank's token-slots routed to e            (FSEP == FSDP)
  dWg   = per rank sum_t sum_k dl_tk x_t at row e_k
"""
from __future__ import annotations

import torch


def _rel(a, b):
    a = a.float()
    b = b.float()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def layer_ref(xs, dys, wg, expert_weights, idx_l, w_l, on_expert=None):
    """xs/dys: per-rank [T, H] cuda tensors (bf16 values); wg [E, H];
    expert_weights(e) -> (w1 [F, H], w3 [F, H], w2 [H, F]) cuda tensors;
    idx_l / w_l: per-rank [T, K] int / float cuda tensors (oracle routing).
    on_expert(e, dW1, dW3, dW2) is called with each expert's fp32 gradient
    (so a caller can compare and free them one expert at a time).
    Returns (ys, dxs, dWgs): per-rank fp32 tensors."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        E = wg.shape[0]
        N = len(xs)
        xf = [x.float() for x in xs]
        dyf = [d.float() for d in dys]
        ys = [torch.zeros_like(x) for x in xf]
        dxs = [torch.zeros_like(x) for x in xf]
        dws = [torch.zeros(i.shape, device=i.device, dtype=torch.float32) for i in idx_l]
        for e in range(E):
            w1, w3, w2 = (t.float() for t in expert_weights(e))
            dW1 = torch.zeros_like(w1)
            dW3 = torch.zeros_like(w3)
            dW2 = torch.zeros_like(w2)
            for i in range(N):
                t, k = torch.nonzero(idx_l[i] == e, as_tuple=True)
                if t.numel() == 0:
                    continue
                xe = xf[i][t]
                g = xe @ w1.t()
                u = xe @ w3.t()
                sg = torch.sigmoid(g)
                a = g * sg * u
                ye = a @ w2.t()
                we = w_l[i][t, k][:, None]
                ys[i].index_add_(0, t, we * ye)
                dws[i][t, k] = (dyf[i][t] * ye).sum(1)
                dye = we * dyf[i][t]
                da = dye @ w2
                du = da * g * sg
                dg = da * u * sg * (1.0 + g * (1.0 - sg))
                dxs[i].index_add_(0, t, dg @ w1 + du @ w3)
                dW2 += dye.t() @ a
                dW1 += dg.t() @ xe
                dW3 += du.t() @ xe
                del g, u, sg, a, ye, dye, da, du, dg, xe
            if on_expert is not None:
                on_expert(e, dW1, dW3, dW2)
            del dW1, dW3, dW2
        dWgs = []
        wgf = wg.float()
        for i in range(N):
            w = w_l[i]
            dl = w * (dws[i] - (w * dws[i]).sum(1, keepdim=True))
            dWg = torch.zeros(E, xf[i].shape[1], device=xf[i].device)
            for k in range(idx_l[i].shape[1]):
                dxs[i] += dl[:, k:k + 1] * wgf[idx_l[i][:, k]]
                dWg.index_add_(0, idx_l[i][:, k], dl[:, k:k + 1] * xf[i])
            dWgs.append(dWg)
        return ys, dxs, dWgs
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
