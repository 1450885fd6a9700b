"""Multi-GPU host driver: one process per GPU, torch.distributed for plumbing.

Two partitionings:

* Materialised fills (configs C1-C4) shard contiguous index ranges; rank r
  owns [first + r*n/G, first + (r+1)*n/G) and writes its slab of the
  row-major array through the fill's `first_index`. No collective: the points
  stay resident on their GPU (`index_shard`).
* The fused render (config C5) splits the image into row bands; every pixel
  is computed by exactly one GPU with the single-GPU summation order, so the
  gathered image is bit-identical to the 1-GPU render. One collective — an
  all-gather of the fp32 bands (NCCL over NVLink on a GPU box, gloo in the
  CPU tests) — assembles the image (`render_distributed`).

* Integration (quality.cpp:214-282) splits the fixed 4096-index chunks into
  contiguous rank ranges; the Kahan chunk partials are all-gathered and
  combined by reduce_deterministic in chunk order (or the exact int64 sums
  all-reduced), so the estimate is bit-identical to the single-GPU one
  (`integrate_distributed`).
* The paper's own split (`partition_by_extra_dimension`,
  imageplane.cpp:114-130): every GPU renders ALL pixels but only its residue
  class of samples, i == rev_2(rank) (mod world), into int64 accumulators;
  one NCCL all-reduce(sum) and a finalize give an image bit-identical to the
  single-GPU int render, because the int accumulator is exactly associative
  (`render_distributed_samples`).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def index_shard(first: int, n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous index range [start, start + count) of `rank` (balanced)."""
    lo = first + n * rank // world
    hi = first + n * (rank + 1) // world
    return lo, hi - lo


def row_bands(height: int, world: int):
    """Row bands [(r0, r1)] per rank, sizes differing by at most one row."""
    return [(height * r // world, height * (r + 1) // world) for r in range(world)]


def render_distributed_samples(width: int, height: int, spp: int,
                               kind: str = "pixel-shifted-lattice", seed: int = 0, group=None,
                               partial_renderer: Optional[Callable] = None,
                               finalize: Optional[Callable] = None) -> torch.Tensor:
    """Sample-partitioned int render across ranks (world a power of two).

    `partial_renderer(part, parts) -> int64 [height, width]` and
    `finalize(acc, spp) -> float32 image` default to the CUDA kernels
    (qmc_render_partial / qmc_render_finalize); tests inject CPU stand-ins."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if partial_renderer is None:
        from . import render_partial

        acc = render_partial(width, height, spp, rank, world, kind=kind, seed=seed)
    else:
        acc = partial_renderer(rank, world)
    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)  # exact int64 sum
    if finalize is None:
        from . import render_finalize

        return render_finalize(acc, spp)
    return finalize(acc, spp)


def sample_partition(part: int, parts: int, base: int = 2) -> Tuple[int, int]:
    """(remainder, modulus) of the indices owned by `part` (imageplane.cpp:114-130)."""
    from . import partition_by_extra_dimension

    return partition_by_extra_dimension(part, parts, base)


def gather_bands(band: torch.Tensor, height: int, width: int, group=None) -> torch.Tensor:
    """All-gather the per-rank row bands into the full [height, width] image.

    Bands are padded to the largest band so one all_gather_into_tensor moves
    everything in a single collective."""
    world = dist.get_world_size(group)
    bands = row_bands(height, world)
    rows = max(r1 - r0 for r0, r1 in bands)
    if all(r1 - r0 == rows for r0, r1 in bands):
        # equal bands (height divisible by the world size, e.g. 2160 rows on
        # 1/2/4/8 GPUs): the collective writes the image itself, no pad or cat
        full = torch.empty((height, width), dtype=band.dtype, device=band.device)
        dist.all_gather_into_tensor(full, band.contiguous(), group=group)
        return full
    pad = torch.zeros((rows, width), dtype=band.dtype, device=band.device)
    pad[: band.shape[0]] = band
    full = torch.empty((world * rows, width), dtype=band.dtype, device=band.device)
    dist.all_gather_into_tensor(full, pad, group=group)
    parts = [full[r * rows: r * rows + (r1 - r0)] for r, (r0, r1) in enumerate(bands)]
    return torch.cat(parts, 0)


def render_distributed(width: int, height: int, spp: int, kind: str = "pixel-shifted-lattice",
                       accum: str = "kahan", seed: int = 0, group=None,
                       band_renderer: Optional[Callable] = None) -> torch.Tensor:
    """Render rank's row band on its GPU, then one all-gather of the bands.

    `band_renderer(r0, r1) -> [r1-r0, width] tensor` defaults to the CUDA
    render (libqmcgpu qmc_render); tests inject a stand-in to exercise the
    partition/gather logic on CPU ranks."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = row_bands(height, world)[rank]
    if band_renderer is None:
        from . import render

        band = render(width, height, spp, kind=kind, accum=accum, seed=seed, rows=(r0, r1))
    else:
        band = band_renderer(r0, r1)
    return gather_bands(band, height, width, group)


def chunk_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Rank's contiguous share [c0, c1) of the ceil(n / 4096) integration chunks."""
    chunks = (n + 4095) // 4096
    return chunks * rank // world, chunks * (rank + 1) // world


def integrate_distributed(kind: str, integrand: str, n: int, dims: int, accum: str = "kahan",
                          group=None, partials_fn: Optional[Callable] = None,
                          reduce_fn: Optional[Callable] = None, **stream_kw) -> float:
    """Multi-rank integrate(): each rank evaluates its chunk range on its GPU
    (qmc_integrate_partials); Kahan partials are gathered to every rank (one
    all-gather of the padded per-rank vectors) and summed in chunk order by
    reduce_deterministic; int sums take one all-reduce. Returns the estimate,
    bit-identical to the single-GPU qmc_integrate. `partials_fn(c0, c1)` and
    `reduce_fn(ranks, values)` default to the CUDA path; tests inject CPU
    stand-ins."""
    import numpy as np

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    c0, c1 = chunk_range(n, world, rank)
    if partials_fn is None:
        from . import integrate_partials

        def partials_fn(a, b):
            return integrate_partials(kind, integrand, n, dims, a, b, accum, **stream_kw)
    if reduce_fn is None:
        from . import reduce_deterministic as reduce_fn
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else \
        torch.device("cpu")
    if accum == "int":
        t = torch.tensor([int(partials_fn(c0, c1))], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)  # exact
        return float(int(t.item())) / 4294967296.0 / n
    mine = np.asarray(partials_fn(c0, c1), np.float64)
    chunks = (n + 4095) // 4096
    width = max(chunks * (r + 1) // world - chunks * r // world for r in range(world))
    pad = torch.zeros(width, dtype=torch.float64, device=dev)
    pad[: mine.size] = torch.from_numpy(mine).to(dev)
    full = torch.empty(world * width, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(full, pad, group=group)
    full = full.cpu().numpy()
    ranks, values = [], []
    for r in range(world):
        a, b = chunk_range(n, world, r)
        ranks.extend(range(a, b))
        values.extend(full[r * width: r * width + (b - a)].tolist())
    return reduce_fn(ranks, values) / n
