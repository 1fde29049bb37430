"""fp64 restatement of the train stage (TEST INFRASTRUCTURE ONLY).

The reference has no model: its trainer is the checksum trainer_step
(pipeline.hpp:103-124), and the paper trains a 3-layer GraphSAGE on the sampled
blocks. This file restates the model the GPU train stage
(paper_2406_13984_b200/csrc/fdg_sage.cu) implements, in numpy float64, so the
GPU's fp32 loss can be checked at 1e-5 relative. Parity for this stage is pinned
to this restatement and to an independent torch formulation
(tests/test_oracle.py::test_sage_oracle_matches_torch), not to the reference.

Blocks follow from sample_khop (sampling.hpp:72-134): every node is expanded at
most once, so node v's sampled in-edges are exactly the edges with dst == v;
layer k = 1..L computes nodes [0, D_{L-k}) with D_j = layer_nodes[j+1].
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    """common.hpp:77-82 on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, np.uint64).copy()
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def labels(nodes: np.ndarray, label_seed: int, classes: int) -> np.ndarray:
    return (splitmix64(np.asarray(nodes, np.uint64) ^ np.uint64(label_seed)) % np.uint64(classes)).astype(np.int64)


def hop_rows(layer_nodes, n_nodes: int, n_layers: int) -> list[int]:
    """D_j, j = 0..L: running max of layer_nodes[0..j+1], capped at n_nodes."""
    ln = [int(v) for v in layer_nodes]
    out = []
    for j in range(n_layers + 1):
        out.append(min(max(ln[: j + 2]) if ln else 0, n_nodes))
    return out


def sage_forward(x: np.ndarray, nodes: np.ndarray, edges: np.ndarray, layer_nodes, weights, label_seed: int):
    """Returns (loss, logits[D_0, C]) in float64. x: [n_nodes, d] rows of X (any float dtype),
    edges: [E, 2] {src_local, dst_local}, weights: [(W_neigh, W_self, b)] per layer."""
    L = len(weights)
    n = len(nodes)
    D = hop_rows(layer_nodes, n, L)
    h = np.asarray(x, np.float64)
    src = np.asarray(edges[:, 0], np.int64) if len(edges) else np.zeros(0, np.int64)
    dst = np.asarray(edges[:, 1], np.int64) if len(edges) else np.zeros(0, np.int64)
    for k in range(1, L + 1):
        rows = D[L - k]
        wn, ws, b = (np.asarray(a, np.float64) for a in weights[k - 1])
        sel = dst < rows
        agg = np.zeros((rows, h.shape[1]))
        np.add.at(agg, dst[sel], h[src[sel]])
        cnt = np.bincount(dst[sel], minlength=rows).astype(np.float64)
        mean = np.divide(agg, cnt[:, None], out=np.zeros_like(agg), where=cnt[:, None] > 0)
        out = mean @ wn + h[:rows] @ ws + b
        h = np.maximum(out, 0.0) if k < L else out
    logits = h
    if len(logits) == 0:
        return 0.0, logits
    y = labels(nodes[: len(logits)], label_seed, logits.shape[1])
    mx = logits.max(axis=1)
    lse = np.log(np.exp(logits - mx[:, None]).sum(axis=1)) + mx
    return float(np.mean(lse - logits[np.arange(len(logits)), y])), logits


def sage_grads(x: np.ndarray, nodes: np.ndarray, edges: np.ndarray, layer_nodes, weights, label_seed: int):
    """(loss, [(dW_neigh, dW_self, db) per layer]) of the same model by torch fp64 autograd:
    the reference for the GPU backward (fdg_sage_backward)."""
    import torch
    L = len(weights)
    D = hop_rows(layer_nodes, len(nodes), L)
    h = torch.tensor(np.asarray(x, np.float64))
    e = torch.tensor(np.asarray(edges, np.int64)).reshape(-1, 2)
    params = [tuple(torch.tensor(np.asarray(a, np.float64), requires_grad=True) for a in w) for w in weights]
    for k in range(1, L + 1):
        rows = D[L - k]
        wn, ws, b = params[k - 1]
        m = e[:, 1] < rows
        s = torch.zeros(rows, h.shape[1], dtype=torch.float64).index_add(0, e[m, 1], h[e[m, 0]])
        c = torch.zeros(rows, dtype=torch.float64).index_add(0, e[m, 1], torch.ones(int(m.sum()), dtype=torch.float64))
        out = (s / c.clamp(min=1).unsqueeze(1)) @ wn + h[:rows] @ ws + b
        h = torch.relu(out) if k < L else out
    y = torch.tensor(labels(nodes[: len(h)], label_seed, h.shape[1]))
    loss = torch.nn.functional.cross_entropy(h, y)
    loss.backward()
    return float(loss.detach()), [tuple(p.grad.numpy() for p in ps) for ps in params]
