"""Multi-GPU y-slab decomposition with depth-T halo exchange.

The padded domain (ny+2, nx+2) is split into `world` contiguous full-width
slabs of interior rows, one per GPU (the reference's full-width row-band
preference, planner.py:230-231). Rank r owns interior rows [y0, y1) and keeps
a local padded grid of its owned rows plus `depth` halo rows on each side
that has a neighbour (the global ghost row on the sides that do not). Every
epoch of s <= depth steps:

  1. local solve: the B200 kernel advances the local grid s steps, treating
     its outermost rows as frozen — exactly the trapezoid argument of
     tile_active_region (planner.py:272-286): after s steps every row at
     distance >= s from a frozen halo edge is exact, so the owned rows are;
  2. exchange: send the first/last `depth` owned rows to the upper/lower
     neighbour, receive its rows into the halo (point-to-point only — a
     5-point stencil needs no collective reduction).

Results are bitwise identical to the single-GPU solve and to
jacobi_reference for any world size (the inter-device analogue of the
worker-count independence the reference tests, test_engine.py:61-77).

The exchange backend is pluggable: torch.distributed point-to-point
(NCCL over NVLink between GPUs; gloo for CPU tests) or in-process virtual
ranks (several slabs on one device, used to check the decomposition on a
single GPU without ranks that wait on each other).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["slab_rows", "SlabGeometry", "SlabSolver", "VirtualSlabs"]


def slab_rows(ny: int, world: int, rank: int) -> tuple[int, int]:
    """Owned interior rows [y0, y1) of `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if ny < world:
        raise ValueError(f"{ny} rows cannot be split over {world} ranks")
    base, rem = divmod(ny, world)
    y0 = rank * base + min(rank, rem)
    return y0, y0 + base + (1 if rank < rem else 0)


@dataclass(frozen=True)
class SlabGeometry:
    nx: int
    ny: int
    world: int
    rank: int
    depth: int

    @property
    def rows(self) -> tuple[int, int]:
        return slab_rows(self.ny, self.world, self.rank)

    @property
    def halo_top(self) -> int:
        """Local rows above the owned rows (the global ghost row for rank 0)."""
        return self.depth if self.rank > 0 else 1

    @property
    def halo_bottom(self) -> int:
        return self.depth if self.rank < self.world - 1 else 1

    @property
    def owned(self) -> int:
        y0, y1 = self.rows
        return y1 - y0

    @property
    def local_ny(self) -> int:
        """Interior rows of the local padded grid (its rows 0 and -1 are frozen)."""
        return self.owned + self.halo_top + self.halo_bottom - 2

    @property
    def global_row0(self) -> int:
        """Padded global row index of local row 0."""
        return self.rows[0] + 1 - self.halo_top

    def validate(self):
        if self.depth < 1:
            raise ValueError("depth must be at least 1")
        # a neighbour's halo must come from the adjacent slab only
        for r in range(self.world):
            y0, y1 = slab_rows(self.ny, self.world, r)
            if self.world > 1 and y1 - y0 < self.depth:
                raise ValueError(f"slab of {y1 - y0} rows is thinner than depth {self.depth}")


class SlabSolver:
    """One rank's slab. `backend` is torch.distributed (already initialised)
    or None for a single rank; `local_solve(src, dst, nx, ny, steps)` advances
    a padded local grid (the B200 kernel on GPU ranks)."""

    def __init__(self, geo: SlabGeometry, local_solve, dist=None, group=None):
        geo.validate()
        self.geo = geo
        self.local_solve = local_solve
        self.dist = dist
        self.group = group
        self.a = None
        self.b = None

    # -- local buffers -------------------------------------------------------
    def load(self, global_padded):
        """Take this rank's rows (owned + halo) from a full padded grid tensor."""
        g = self.geo
        r0 = g.global_row0
        self.a = global_padded[r0:r0 + g.local_ny + 2].clone()
        self.b = self.a.clone()
        return self

    def attach(self, a, b):
        """Use caller-provided local buffers (shape (local_ny+2, pitch))."""
        self.a, self.b = a, b
        return self

    def owned_view(self):
        g = self.geo
        return self.a[g.halo_top:g.halo_top + g.owned]

    # -- one epoch -----------------------------------------------------------
    def exchange_ops(self):
        """(send, recv, peer) triples for this rank's halo exchange."""
        g, a = self.geo, self.a
        ops = []
        ht, own, d = g.halo_top, g.owned, g.depth
        if g.rank > 0:
            ops.append((a[ht:ht + d], a[0:ht], g.rank - 1))
        if g.rank < g.world - 1:
            ops.append((a[ht + own - d:ht + own], a[ht + own:ht + own + d], g.rank + 1))
        return ops

    def exchange(self):
        if self.geo.world == 1:
            return
        d = self.dist
        p2p = []
        for send, recv, peer in self.exchange_ops():
            p2p.append(d.P2POp(d.isend, send.contiguous(), peer, self.group))
            p2p.append(d.P2POp(d.irecv, recv, peer, self.group))
        for req in d.batch_isend_irecv(p2p):
            req.wait()

    def step(self, steps: int):
        g = self.geo
        self.local_solve(self.a, self.b, g.nx, g.local_ny, steps)
        self.a, self.b = self.b, self.a

    def run(self, total_steps: int):
        done = 0
        while done < total_steps:
            s = min(self.geo.depth, total_steps - done)
            self.step(s)
            done += s
            if done < total_steps:
                self.exchange()
        return self


class VirtualSlabs:
    """All `world` slabs of a domain on one device/process: the same epochs,
    with the exchange done by in-process copies (no rank ever waits on
    another's kernel)."""

    def __init__(self, nx: int, ny: int, world: int, depth: int, local_solve):
        self.ranks = [SlabSolver(SlabGeometry(nx, ny, world, r, depth), local_solve)
                      for r in range(world)]

    def load(self, global_padded):
        for s in self.ranks:
            s.load(global_padded)
        return self

    def exchange(self):
        sends = {}
        for s in self.ranks:
            for send, recv, peer in s.exchange_ops():
                sends[(s.geo.rank, peer)] = send.clone()
        for s in self.ranks:
            for send, recv, peer in s.exchange_ops():
                recv.copy_(sends[(peer, s.geo.rank)])

    def run(self, total_steps: int):
        depth = self.ranks[0].geo.depth
        done = 0
        while done < total_steps:
            k = min(depth, total_steps - done)
            for s in self.ranks:
                s.step(k)
            done += k
            if done < total_steps:
                self.exchange()
        return self

    def gather(self, out):
        """Write every rank's owned rows into a full padded grid `out`."""
        for s in self.ranks:
            y0, y1 = s.geo.rows
            out[y0 + 1:y1 + 1] = s.owned_view()
        return out
