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
