"""CPU multi-process (gloo, world_size 2) tests of the head-sharded layer.

The GPU runs use the same helpers over NCCL (bench.py under torchrun).  Here
each rank computes its heads' attention with the CPU oracle (test
infrastructure) so that the sharding + exchange logic is checked end to end:
the dynamic-mode mask is built only on the scoring rank and broadcast, and
the gathered head shards equal the single-process result.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_20470_b200.sharding import (broadcast_mask, broadcast_scoring_features,
                                            gather_heads, head_shards, or_allgather_mask,
                                            score_rank)


def test_head_shards_cover_all_heads():
    for H in (1, 2, 5, 24, 40):
        for world in range(1, min(H, 8) + 1):
            sh = head_shards(H, world)
            assert sum(n for _, n in sh) == H
            assert [h for h, _ in sh] == list(np.cumsum([0] + [n for _, n in sh])[:-1])
            assert max(n for _, n in sh) - min(n for _, n in sh) <= 1
    assert head_shards(40, 8) == [(5 * r, 5) for r in range(8)]
    assert head_shards(24, 8) == [(3 * r, 3) for r in range(8)]
    with pytest.raises(ValueError):
        head_shards(2, 3)
    assert score_rank(24, 8, 2) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle
    P = pyoracle.port()
    nf, nt, bs, H, d = 4, 64, 16, 4, 8
    S = nf * nt
    q, k, v = P.random_batch(S, H, d, 11, threads=1)
    cfg = pyoracle.Cfg(1, 1.4, 0.7, 1e-6, 0.5, 0.3, 0.0, 0.3)
    nb = (S + bs - 1) // bs
    mask = torch.zeros((nb, (nb + 7) // 8), dtype=torch.uint8)
    if rank == score_rank(H, world, 2):
        # only the rank holding heads 0..H_f-1 scores the layer
        mask[:] = torch.from_numpy(P.build_mask(nf, nt, bs, cfg, 7, False, q[:, :2].copy(),
                                                k[:, :2].copy()))
    broadcast_mask(mask, src=0)
    h0, n = head_shards(H, world)[rank]
    sl = slice(h0, h0 + n)
    out = P.masked_attention_exact(nf, nt, bs, mask.numpy(), q[:, sl].copy(), k[:, sl].copy(),
                                   v[:, sl].copy())
    full = gather_heads(torch.from_numpy(out), H)
    np.save(os.path.join(result_dir, f"r{rank}.npy"), full.numpy())
    np.save(os.path.join(result_dir, f"m{rank}.npy"), mask.numpy())
    dist.destroy_process_group()


def test_sharded_dynamic_layer_gloo(tmp_path, port):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    P = port
    nf, nt, bs, H, d = 4, 64, 16, 4, 8
    q, k, v = P.random_batch(nf * nt, H, d, 11, threads=1)
    cfg = pytest.importorskip("oracle.pyoracle").Cfg(1, 1.4, 0.7, 1e-6, 0.5, 0.3, 0.0, 0.3)
    mask = P.build_mask(nf, nt, bs, cfg, 7, False, q[:, :2].copy(), k[:, :2].copy())
    want = P.masked_attention_exact(nf, nt, bs, mask, q, k, v)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"m{r}.npy"), mask)
        assert np.array_equal(np.load(tmp_path / f"r{r}.npy"), want)


def _split_worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S, H, d, nb = 96, 4, 8, 13
    g = torch.Generator().manual_seed(5)
    q = torch.randn(S, H, d, generator=g) + rank  # only rank 0's copy is authoritative
    k = torch.randn(S, H, d, generator=g) - rank
    qs, ks = broadcast_scoring_features(q, k, 2, src=0)
    # partial masks: common base bits + this rank's share of the scored bits
    rng = np.random.default_rng(9)
    base = rng.integers(0, 256, (nb, 2), dtype=np.uint8) & 0x11
    scored = rng.integers(0, 256, (nb, 2), dtype=np.uint8) & 0xEE
    mine = scored & (np.uint8(0x0F) if rank == 0 else np.uint8(0xF0))
    mask = torch.from_numpy(base | mine)
    or_allgather_mask(mask)
    np.save(os.path.join(result_dir, f"q{rank}.npy"), qs.numpy())
    np.save(os.path.join(result_dir, f"k{rank}.npy"), ks.numpy())
    np.save(os.path.join(result_dir, f"m{rank}.npy"), mask.numpy())
    np.save(os.path.join(result_dir, "want.npy"), base | scored)
    dist.destroy_process_group()


def test_split_scoring_exchange_gloo(tmp_path):
    """Split dynamic scoring (SURVEY 8e option 2): the H_f scoring heads are
    broadcast from the rank that holds them, and the per-rank partial masks
    are OR-combined identically on every rank."""
    world = 2
    mp.spawn(_split_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g = torch.Generator().manual_seed(5)
    q = torch.randn(96, 4, 8, generator=g)
    k = torch.randn(96, 4, 8, generator=g)
    want = np.load(tmp_path / "want.npy")
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"q{r}.npy"), q[:, :2].numpy())
        assert np.array_equal(np.load(tmp_path / f"k{r}.npy"), k[:, :2].numpy())
        assert np.array_equal(np.load(tmp_path / f"m{r}.npy"), want)
