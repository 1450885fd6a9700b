"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): index-range shards
cover the sequence exactly once, and the row-band all-gather reassembles the
image the single-process render produces (bands from the oracle)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_15584_b200.distributed import index_shard, row_bands


def test_index_shards_partition():
    for first, n, world in [(0, 1 << 28, 8), (5, 1001, 3), (7, 3, 4)]:
        spans = [index_shard(first, n, world, r) for r in range(world)]
        assert spans[0][0] == first
        for (a, c), (b, _) in zip(spans, spans[1:]):
            assert a + c == b
        assert sum(c for _, c in spans) == n


def test_row_bands():
    for h, w in [(2160, 8), (5, 3), (1, 2)]:
        b = row_bands(h, w)
        assert b[0][0] == 0 and b[-1][1] == h
        assert all(r1 - r0 in (h // w, h // w + 1) for r0, r1 in b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, w, h, spp, expect_path, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_15584_b200.distributed import render_distributed

    full = torch.from_numpy(np.load(expect_path))
    img = render_distributed(w, h, spp, band_renderer=lambda r0, r1: full[r0:r1].clone())
    if rank == 0:
        np.save(out_path, img.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_render_band_gather_gloo(tmp_path, oracle, columns64, world):
    from oracle import ptr

    w, h, spp = 40, 23, 4
    img = np.zeros((h, w), np.float32)
    cols2 = np.ascontiguousarray(columns64[:2])
    assert oracle.qo_render(w, h, spp, 4, 0, 0, ptr(cols2), ptr(img)) == 0
    exp_path, out_path = str(tmp_path / "exp.npy"), str(tmp_path / "out.npy")
    np.save(exp_path, img)
    mp.spawn(_worker, args=(world, _free_port(), w, h, spp, exp_path, out_path), nprocs=world,
             join=True)
    np.testing.assert_array_equal(np.load(out_path), img)


def _worker_samples(rank, world, port, w, h, spp, cols_path, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import load_oracle, ptr
    from paper_2307_15584_b200 import partition_by_extra_dimension  # noqa: F401
    from paper_2307_15584_b200.distributed import render_distributed_samples

    o = load_oracle()
    cols2 = np.load(cols_path)

    def partial(part, parts):
        # residue class of part: i == rev_2(part) (mod parts)
        rem = int("{:0{w}b}".format(part, w=parts.bit_length() - 1)[::-1] or "0", 2)
        acc = np.zeros((h, w), np.int64)
        assert o.qo_render_partial_int(w, h, spp, 4, 0, ptr(cols2), rem, parts, ptr(acc)) == 0
        return torch.from_numpy(acc)

    def finalize(acc, s):
        return torch.from_numpy(
            ((acc.numpy().astype(np.float64) / 4294967296.0) / s).astype(np.float32))

    img = render_distributed_samples(w, h, spp, partial_renderer=partial, finalize=finalize)
    if rank == 0:
        np.save(out_path, img.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_render_sample_partition_gloo(tmp_path, oracle, columns64, world):
    """The paper's sample partition (i == rev_2(rank) mod world): int64
    partials + one all-reduce reproduce the single-process int render."""
    from oracle import ptr

    w, h, spp = 24, 17, 12
    cols2 = np.ascontiguousarray(columns64[:2])
    full = np.zeros((h, w), np.float32)
    assert oracle.qo_render(w, h, spp, 4, 1, 0, ptr(cols2), ptr(full)) == 0
    cols_path, out_path = str(tmp_path / "c.npy"), str(tmp_path / "o.npy")
    np.save(cols_path, cols2)
    mp.spawn(_worker_samples, args=(world, _free_port(), w, h, spp, cols_path, out_path),
             nprocs=world, join=True)
    np.testing.assert_array_equal(np.load(out_path), full)


def _worker_integrate(rank, world, port, n, accum, vals_path, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_15584_b200.distributed import integrate_distributed

    vals = np.load(vals_path)  # stand-in chunk partials (kahan) / chunk int sums (int)

    def partials(c0, c1):
        return vals[c0:c1] if accum == "kahan" else int(vals[c0:c1].astype(np.int64).sum())

    est = integrate_distributed("sobol", "product-sine", n, 4, accum, partials_fn=partials)
    if rank == 0:
        np.save(out_path, np.array([est]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("accum", ["kahan", "int"])
def test_integrate_distributed_gloo(tmp_path, world, accum):
    """Chunk ranges per rank + one all-gather and the rank-ordered
    reduce_deterministic (or one int all-reduce) reproduce the single-process
    combine exactly."""
    import paper_2307_15584_b200 as q

    n = 4096 * 37 + 5
    chunks = (n + 4095) // 4096
    rng = np.random.default_rng(world)
    if accum == "kahan":
        vals = rng.standard_normal(chunks) * 10.0 ** rng.integers(-8, 8, chunks)
        exp = q.reduce_deterministic(np.arange(chunks), vals) / n
    else:
        vals = rng.integers(-2**40, 2**40, chunks).astype(np.float64)
        exp = float(int(vals.astype(np.int64).sum())) / 4294967296.0 / n
    vp, op = str(tmp_path / "v.npy"), str(tmp_path / "o.npy")
    np.save(vp, vals)
    mp.spawn(_worker_integrate, args=(world, _free_port(), n, accum, vp, op), nprocs=world,
             join=True)
    assert np.load(op)[0] == exp
