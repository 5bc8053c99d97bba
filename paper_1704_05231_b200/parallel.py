"""Multi-GPU work partitioning (one process per GPU; no data-path collective).

The path shards into independent units:

* batched banks (config 3): images, contiguous blocks per rank;
* large single-image banks (config 5): (frequency i, direct orientation k)
  units -- unit id i*(N/2+1)+k, computing theta_k and, when it exists,
  pi-theta_k from the same row pass (bank.py:109-116) -- split into
  contiguous runs per rank by an exact linear partition over a device-time
  model measured on the B200 (partition_units);
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


# Device-time model of the bank kernels, fitted to the B200 measurements in
# profiles/r02/unit_costs_c5.json (tools/unit_costs.py: every contiguous k-range of every
# config-5 frequency, kernel time from the live profile).  Per frequency of half-width
# h = ceil(r sigma), computing g directs of which `single` have one output (theta = 0, pi/2)
# and `double` two (theta, pi - theta):
#     cost = A(h) + B1(h) * single + B2(h) * double          (ms on the fit's 8192^2 image)
# with (A, B1, B2) interpolated linearly in h between the fitted half-widths: h = 6 / 12 / 24 / 48 the
# fused tensor-core kernel (bank_umma.cu), h = 96 the tensor-core row + column passes (row_umma.cu,
# col_umma.cu).  Fitted by tools/fit_unit_costs.py (median error 3 %, 90th percentile 9 %; the ranges measured first, on a cold
# GPU, sit up to 45 % below the fit); B1 / B2 then raised by 0.066 / 0.034 / 0.031 / 0.016 / 0.015 ms per unit
# (h = 6 .. 96): what each rank's share, timed as a whole call with a cold L2 in round robin
# (tools/partition_balance.py), took beyond the sum of its kernel times.
# mgpu.cu restates it (same anchors, same order).
_MPX = 67.108864  # the fit's 8192^2 image
_FIT = ((6, 0.0553, 0.2141, 0.3204), (12, 0.0329, 0.2401, 0.3043), (24, 0.0701, 0.2338, 0.2985),
        (48, 0.0638, 0.2936, 0.3483), (96, 0.1561, 0.4585, 0.5044))


def _fit_at(h: int) -> tuple[float, float, float]:
    if h <= _FIT[0][0]:
        return _FIT[0][1:]
    for (h0, *p0), (h1, *p1) in zip(_FIT, _FIT[1:]):
        if h <= h1:
            w = (h - h0) / (h1 - h0)
            return tuple(a + w * (b - a) for a, b in zip(p0, p1))
    return _FIT[-1][1:]


def run_cost(sigma: float, ks, n: int, radius: float = 3.0, mpx: float = 1.0) -> float:
    """Modelled device ms of one rank computing the direct orientations ``ks`` of
    one frequency (one launch for all of them) on an image of ``mpx`` megapixels."""
    ks = list(ks)
    if not ks:
        return 0.0
    h = max(1, math.ceil(radius * sigma))
    a, b1, b2 = _fit_at(h)
    single = sum(1 for k in ks if k == 0 or 2 * k == n)
    return mpx / _MPX * (a + b1 * single + b2 * (len(ks) - single))


def bank_unit_costs(freqs, sigmas, n: int, radius: float = 3.0) -> dict[int, float]:
    """Modelled device cost of every (frequency i, direct k) unit computed alone
    (unit id i*(N/2+1)+k; theta = 0 has no B term, theta = pi/2 a real J)."""
    nh = n // 2
    return {i * (nh + 1) + k: run_cost(s, [k], n, radius) for i, s in enumerate(sigmas) for k in range(nh + 1)}


def partition_units(freqs, sigmas, n: int, world: int, radius: float = 3.0) -> list[list[int]]:
    """Split the bank's (frequency, direct k) units over ``world`` ranks as
    contiguous runs of the sequence ordered by frequency (largest sigma first)
    then k, minimising the largest modelled rank cost (exact linear-partition
    DP).  Contiguity keeps a rank's directs of one frequency together so they
    share one launch (and its fixed cost); a plain LPT over single units
    splits frequencies across ranks."""
    nh = n // 2
    order = [(i, k) for i in sorted(range(len(sigmas)), key=lambda i: (-sigmas[i], i)) for k in range(nh + 1)]
    m = len(order)
    world = max(1, min(world, m))

    def seg_cost(a, b):  # units order[a:b]
        return partition_cost([[i * (nh + 1) + k for i, k in order[a:b]]], sigmas, n, radius)[0]

    cost = [[0.0] * (m + 1) for _ in range(m + 1)]
    for a in range(m):
        for b in range(a + 1, m + 1):
            cost[a][b] = seg_cost(a, b)
    inf = float("inf")
    best = [[inf] * (m + 1) for _ in range(world + 1)]
    cut = [[0] * (m + 1) for _ in range(world + 1)]
    best[0][0] = 0.0
    for r in range(1, world + 1):
        for b in range(1, m + 1):
            for a in range(r - 1, b):
                v = max(best[r - 1][a], cost[a][b])
                if v < best[r][b]:
                    best[r][b], cut[r][b] = v, a
    bounds, b = [], m
    for r in range(world, 0, -1):
        a = cut[r][b]
        bounds.append((a, b))
        b = a
    bounds.reverse()
    parts = [sorted(i * (nh + 1) + k for i, k in order[a:b]) for a, b in bounds]
    return _refine(parts, sigmas, n, radius)


def _refine(parts, sigmas, n: int, radius: float, rounds: int = 200):
    """Local search on the partition: move a unit off the most loaded rank, or
    swap it with another rank's unit, while that lowers the larger of the two
    ranks' costs below the current maximum (deterministic; ends at a local
    optimum)."""
    parts = [list(p) for p in parts]
    cost = partition_cost(parts, sigmas, n, radius)

    def c1(p):
        return partition_cost([p], sigmas, n, radius)[0]

    for _ in range(rounds):
        r = max(range(len(parts)), key=lambda j: (cost[j], -j))
        top, best = cost[r], None
        for u in parts[r]:
            ru = [x for x in parts[r] if x != u]
            for q in range(len(parts)):
                if q == r:
                    continue
                cand = [(c1(ru), c1(parts[q] + [u]), ru, parts[q] + [u])]
                for v in parts[q]:
                    qv = [x for x in parts[q] if x != v] + [u]
                    cand.append((c1(ru + [v]), c1(qv), ru + [v], qv))
                for a, b, pa, pb in cand:
                    m = max(a, b)
                    if m < top - 1e-12 and (best is None or m < best[0] - 1e-12):
                        best = (m, q, a, b, pa, pb)
        if best is None:
            break
        _, q, a, b, pa, pb = best
        parts[r], parts[q], cost[r], cost[q] = pa, pb, a, b
    return [sorted(p) for p in parts]


def partition_cost(parts, sigmas, n: int, radius: float = 3.0) -> list[float]:
    """Modelled cost of each rank's unit list (row launches shared per frequency)."""
    nh = n // 2
    out = []
    for p in parts:
        runs: dict[int, list[int]] = {}
        for u in p:
            runs.setdefault(u // (nh + 1), []).append(u % (nh + 1))
        c = 0.0  # fixed summation order (frequency, then k) -- mgpu.cu sums the same way
        for i in sorted(runs):
            c += run_cost(sigmas[i], sorted(runs[i]), n, radius)
        out.append(c)
    return out


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
    units = partition_units(spec.frequencies, sig, spec.orientations_n, world, radius)[rank]
    if compute is None:
        from .device import compute_bank as compute_dev

        def compute(im, sp, kd, un):
            return compute_dev(im, sp, kd, True, un)[0]
    out = compute(img, spec, kind, units)
    return out, unit_entries(units, spec.orientations_n)


class LibComm:
    """The C ABI's own multi-GPU driver (fgb_mgpu_*, csrc/mgpu.cu): one process
    per GPU, libfgb200 owns the NCCL communicator; the 128-byte NCCL id is
    shared over ``torch.distributed`` (any backend).  ``bank`` / ``sdft``
    broadcast rank 0's device image (one ncclBroadcast) and compute this
    rank's partition -- the same partition as ``partition_units`` /
    ``sdft_heads`` (restated in C++; a CPU test checks they agree)."""

    def __init__(self, world: int, rank: int, device: int, group=None):
        import ctypes as C

        from . import _native as N

        self.N, self.C = N, C
        self.world, self.rank = world, rank
        idb = (C.c_ubyte * N.FGB_MGPU_ID_BYTES)()
        if rank == 0:
            N.check(N.lib.fgb_mgpu_unique_id(idb), mgpu=True)
        if world > 1:
            import torch.distributed as dist

            obj = [bytes(idb) if rank == 0 else None]
            dist.broadcast_object_list(obj, 0, group=group)
            idb = (C.c_ubyte * N.FGB_MGPU_ID_BYTES).from_buffer_copy(obj[0])
        N.check(N.lib.fgb_mgpu_init(idb, world, rank, device), mgpu=True)

    def units(self, desc) -> list[int]:
        buf = (self.C.c_int32 * 4096)()
        n = self.N.check(self.N.lib.fgb_mgpu_bank_units(self.C.byref(desc), self.world, self.rank, buf, 4096), mgpu=True)
        return list(buf[:n])

    def bank(self, desc, img, out, stream=0):
        self.N.check(self.N.lib.fgb_mgpu_bank(self.C.byref(desc), self.C.c_void_p(img.data_ptr()),
                                              self.C.c_void_p(out.data_ptr()), self.C.c_void_p(stream)), mgpu=True)

    def sdft(self, desc, img, out, stream=0):
        self.N.check(self.N.lib.fgb_mgpu_sdft(self.C.byref(desc), self.C.c_void_p(img.data_ptr()),
                                              self.C.c_void_p(out.data_ptr()), self.C.c_void_p(stream)), mgpu=True)

    def close(self):
        self.N.lib.fgb_mgpu_finalize()
