"""ZeRO-1 data parallelism on CPU.

* partition shapes: shard = ceil(P/N) (64-element aligned), state bytes / rank
* the lockstep bus simulator (oracle interp, rank-order reductions) vs a single
  device on the concatenated batch: fp32 SGD within 1e-5 max abs,
  bf16 Adam within tolerance
* a real 2-process run over torch.distributed (gloo) whose collectives go
  through the same graph: bit-identical to the bus simulation.
"""
import os

import numpy as np
import pytest

from oracle.interp_py import Interp, World
from paper_2303_04759_b200.session import ModelConfig, graph_info, graph_text, synthetic_batch

SMALL = dict(kind="bert", L=1, H=64, A=2, F=128, V=256, S=32, B=2, p=0.0)


def cfg(**kw):
    return ModelConfig(**{**SMALL, **kw})


def batches(c: ModelConfig, n: int, seed: int):
    """n per-rank batches with every position labelled (equal valid counts per
    rank, so the mean of rank means equals the global mean)."""
    ids = np.stack([synthetic_batch(c, seed=seed * 100 + r)[0] for r in range(n)])
    return ids, ids.copy()


@pytest.mark.parametrize("n", [2, 3, 4])
def test_zero_partition_shapes(n):
    c1 = graph_info(cfg(dtype="bf16", opt="adam"))
    cn = graph_info(cfg(dtype="bf16", opt="adam", world=n))
    assert cn["P"] == c1["P"]
    assert cn["P_pad"] % (64 * n) == 0 and cn["P_pad"] >= cn["P"]
    bk = buckets(cfg(dtype="bf16", opt="adam", world=n))
    shard = sum(sh for _, _, sh in bk)
    # every bucket is split into N equal slices of ceil(numel / N)
    assert all(sh == -(-nb // n) for _, nb, sh in bk)
    assert sum(nb for _, nb, _ in bk) == cn["P_pad"]
    # optimizer state (params, m, v) per rank is exactly one shard each
    full_state = c1["state_bytes"] - 3 * c1["P_pad"] * 4
    part_state = cn["state_bytes"] - 3 * shard * 4
    # the bf16 compute copy is sharded too (all-gathered at the top of the step)
    assert part_state - full_state == shard * 2 - c1["P_pad"] * 2


def buckets(c: ModelConfig):
    """ZeRO bucket table (offset, numel, shard) of the step graph"""
    return [tuple(int(x) for x in line.split()) for line in graph_text(c, "buckets").splitlines()]


def unshard(c: ModelConfig, shards, P_pad: int) -> np.ndarray:
    """flat [P_pad] vector from the per-rank shards: rank r holds slice r of
    every bucket, bucket after bucket"""
    out = np.zeros(P_pad, shards[0].dtype)
    so = 0
    for o, n, sh in buckets(c):
        for r, x in enumerate(shards):
            k = min(sh, n - r * sh)
            if k > 0:
                out[o + r * sh:o + r * sh + k] = x[so:so + k]
        so += sh
    return out


def _single_vs_world(c1: ModelConfig, cn: ModelConfig, n: int, steps: int):
    single = Interp(c1.cfg_string(model_only=True))
    world = World(cn.cfg_string(model_only=True), n)
    ls, lw = [], []
    for k in range(steps):
        ids, labels = batches(cn, n, k)
        ls.append(single.step(ids.reshape(-1), labels.reshape(-1)))
        lw.append(world.step(ids, labels))
    P = graph_info(c1)["P"]
    Pn = graph_info(cn)["P_pad"]
    shard = sum(sh for _, _, sh in buckets(cn))
    p_single = single.read("params", P)
    p_world = unshard(cn, [world.read(r, "params", shard) for r in range(n)], Pn)[:P]
    return np.array(ls), np.array(lw), p_single, p_world, world


@pytest.mark.parametrize("n", [2, 4])
def test_world_sgd_fp32_matches_single_device(n):
    """N-rank ZeRO SGD on the split batch == single device on the
    full batch within 1e-5 max abs error."""
    c1 = cfg(B=2 * n, dtype="f32", opt="sgd", lr=0.05)
    cn = cfg(B=2, dtype="f32", opt="sgd", lr=0.05, world=n)
    ls, lw, ps, pw, _ = _single_vs_world(c1, cn, n, steps=4)
    assert np.allclose(lw.mean(axis=1), ls, atol=1e-5)
    assert np.max(np.abs(ps - pw)) <= 1e-5


def test_world_adam_bf16_matches_single_device():
    n = 2
    c1 = cfg(B=4, dtype="bf16", opt="adam", lr=1e-3)
    cn = cfg(B=2, dtype="bf16", opt="adam", lr=1e-3, world=n)
    ls, lw, ps, pw, _ = _single_vs_world(c1, cn, n, steps=3)
    assert np.max(np.abs(lw.mean(axis=1) - ls)) < 1e-2
    # Adam normalises each update to ~lr, so a rounding-level gradient
    # difference near zero can move a parameter by at most ~2 lr per step
    assert np.max(np.abs(ps - pw)) <= 2 * 1e-3 * 3 + 1e-6
    assert np.mean(np.abs(ps - pw) < 1e-6) > 0.99


def test_bus_is_deterministic():
    cn = cfg(B=2, dtype="f32", opt="sgd", lr=0.05, world=3)
    outs = []
    for _ in range(2):
        w = World(cn.cfg_string(model_only=True), 3)
        ids, labels = batches(cn, 3, 7)
        w.step(ids, labels)
        sh = sum(x for _, _, x in buckets(cn))
        outs.append(np.concatenate([w.read(r, "params", sh) for r in range(3)]))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


def test_single_rank_refuses_collectives_without_bus():
    cn = cfg(B=2, dtype="f32", opt="sgd", world=2)
    it = Interp(cn.cfg_string(model_only=True), rank=0)
    ids, labels = batches(cn, 1, 0)
    with pytest.raises(RuntimeError, match="simulation bus"):
        it.step(ids[0], labels[0])


# --------------------------------------------------------- 2 processes, gloo
def _gloo_rank(rank, world, port, cfg_string, steps, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = ModelConfig(**{**SMALL, "B": 2, "dtype": "f32", "opt": "sgd", "lr": 0.05, "world": world})

    def coll(kind, inp, out, w, r):
        t = torch.from_numpy(inp.copy())
        if kind == 0:  # reduce_scatter(sum): all_reduce then keep shard r (zero padded)
            full = torch.zeros(out.size * w)
            full[: t.numel()] = t
            dist.all_reduce(full)
            out[:] = full[r * out.size:(r + 1) * out.size].numpy()
        elif kind == 1:  # all_gather
            parts = [torch.empty_like(t) for _ in range(w)]
            dist.all_gather(parts, t)
            out[:] = torch.cat(parts)[: out.size].numpy()
        else:
            dist.all_reduce(t)
            out[:] = t.numpy()

    it = Interp(cfg_string, rank=rank)
    losses = []
    for k in range(steps):
        ids, labels = batches(c, world, k)
        losses.append(it.step(ids[rank], labels[rank], coll=coll))
    shard = sum(sh for _, _, sh in buckets(c))
    np.save(out_path + f".{rank}.npy", np.concatenate([it.read("params", shard), np.array(losses, np.float32)]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_process_matches_bus(tmp_path):
    import socket

    import torch.multiprocessing as mp
    world, steps = 2, 2
    c = cfg(B=2, dtype="f32", opt="sgd", lr=0.05, world=world)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "rank")
    mp.start_processes(_gloo_rank, args=(world, port, c.cfg_string(model_only=True), steps, out), nprocs=world,
                       join=True, start_method="spawn")
    bus = World(c.cfg_string(model_only=True), world)
    bl = []
    for k in range(steps):
        ids, labels = batches(c, world, k)
        bl.append(bus.step(ids, labels))
    shard = sum(sh for _, _, sh in buckets(c))
    for r in range(world):
        got = np.load(out + f".{r}.npy")
        ref = np.concatenate([bus.read(r, "params", shard), np.array([x[r] for x in bl], np.float32)])
        # two-rank sums are commutative, so gloo's all-reduce order cannot differ
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
