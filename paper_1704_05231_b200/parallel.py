"""Multi-GPU work partitioning (one process per GPU; no data-path collective).

The path shards into independent units:

* batched banks (config 3): images, contiguous blocks per rank;
* large single-image banks (config 5): (frequency i, direct orientation k)
  units -- unit id i*(N/2+1)+k, computing theta_k and, when it exists,
  pi-theta_k from the same row pass (bank.py:109-116) -- balanced by LPT on
  their FLOP cost;
* the localized SDFT (config 4): conjugate u-pairs {u, M-u}; the pair (0, M/2)
  self-pairs are merged so that every shard holds 2*M bins when possible.

The image is broadcast once (``torch.distributed.broadcast`` over NCCL /
NVLink); each rank writes only its own outputs.  These functions are pure
host logic and are tested with gloo on CPU (tests/test_parallel.py).
"""

from __future__ import annotations

import math


def shard_images(n_images: int, world: int) -> list[list[int]]:
    """Contiguous, balanced image blocks per rank."""
    base, extra = divmod(n_images, world)
    out, s = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append(list(range(s, s + n)))
        s += n
    return out


def bank_unit_costs(freqs, sigmas, n: int, radius: float = 3.0) -> dict[int, float]:
    """Relative FP32 cost of every (frequency, direct k) unit.

    Row pass ~ shared FIR over the input (amortised: T per direct), column pass
    4T per emitted pair (2T when theta = 0 has no B term), per pixel.
    """
    nh = n // 2
    costs = {}
    for i, s in enumerate(sigmas):
        t = 2 * max(1, math.ceil(radius * s)) + 1
        for k in range(nh + 1):
            mirror = nh < n - k < n
            col = 2 * t if k == 0 else 4 * t
            costs[i * (nh + 1) + k] = t * 1.2 + col + (0.0 if mirror else 0.0)
    return costs


def lpt_assign(costs: dict[int, float], world: int) -> list[list[int]]:
    """Longest-processing-time-first static assignment; units sorted per rank."""
    loads = [0.0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    for u, c in sorted(costs.items(), key=lambda kv: (-kv[1], kv[0])):
        r = min(range(world), key=lambda j: (loads[j], j))
        parts[r].append(u)
        loads[r] += c
    return [sorted(p) for p in parts]


def sdft_heads(m: int, world: int) -> list[list[int]]:
    """Pair heads u in [0, m/2] per rank (each head owns bins (u,*) and (m-u,*))."""
    heads = list(range(m // 2 + 1))
    # weight: 2 bin rows per head, 1 for the self-paired heads 0 and m/2
    w = {u: (1 if (u == 0 or 2 * u == m) else 2) for u in heads}
    loads = [0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    for u in sorted(heads, key=lambda x: (-w[x], x)):
        r = min(range(world), key=lambda j: (loads[j], j))
        parts[r].append(u)
        loads[r] += w[u]
    return [sorted(p) for p in parts]


def load_balance(parts, costs) -> float:
    """max/mean load of an assignment (1.0 = perfect)."""
    loads = [sum(costs[u] for u in p) for p in parts]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean > 0 else 1.0


def unit_entries(units, n: int) -> list[tuple[int, int]]:
    """(frequency i, orientation k) of every output of a unit list, in the
    compact order the C ABI writes them (fgb_bank_desc.units): per unit its
    direct entry, then the mirror N-k when it exists (bank.py:112-115)."""
    nh = n // 2
    out = []
    for u in units:
        i, k = divmod(u, nh + 1)
        out.append((i, k))
        if nh < n - k < n:
            out.append((i, n - k))
    return out


def head_bins(heads, m: int) -> list[tuple[int, int]]:
    """(u, v) of every bin of a pair-head list in the compact SDFT order."""
    out = []
    for u in heads:
        out += [(u, v) for v in range(m)]
        um = (m - u) % m
        if um != u:
            out += [(um, v) for v in range(m)]
    return out


def sharded_bank(img, spec, kind, group=None, compute=None, radius: float = 3.0):
    """Multi-rank bank of ONE image: rank 0's image is broadcast once
    (torch.distributed over NCCL on B200s, gloo in CPU tests), every rank
    computes its LPT share of (frequency, direct k) units, no collective in
    the data path.  Returns (local outputs [E_local, H, W], entry list).

    ``compute(img, spec, kind, units)`` defaults to the device path
    (paper_1704_05231_b200.device.compute_bank); tests inject a CPU stand-in.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world > 1:
        dist.broadcast(img, 0, group=group)
    sig = [spec.sigma_for(i) for i in range(len(spec.frequencies))]
    costs = bank_unit_costs(spec.frequencies, sig, spec.orientations_n, radius)
    units = lpt_assign(costs, world)[rank]
    if compute is None:
        from .device import compute_bank as compute_dev

        def compute(im, sp, kd, un):
            return compute_dev(im, sp, kd, True, un)[0]
    out = compute(img, spec, kind, units)
    return out, unit_entries(units, spec.orientations_n)
