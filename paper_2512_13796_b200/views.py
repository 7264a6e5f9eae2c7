"""Multi-GPU work partitioning of the render path: one process per
GPU, each with a resident copy of the scene; views are independent units, so no
collective touches the data path.

* ``StaticDealer`` — step s renders views s*world + rank (mod the ring): disjoint per
  step, no coordination at all.
* ``DynamicDealer`` — every rank pulls the next view index from one atomic counter
  (the ``torch.distributed`` store's ``add``, the cross-process analogue of the
  reference's ``parallel_chunks`` work counter, threading.cpp:37-45), so a rank that
  draws cheap views (fewer straddlers) renders more of them.
* ``ShardPlan`` — config 4 (4K): ranks form ``groups`` view groups of ``bands`` image
  bands each; group g renders views g, g + groups, ... and rank (g, b) renders band b
  (``image_bands``) of each of them (strong scaling inside a view, weak across groups).
"""
from dataclasses import dataclass
from typing import List, Optional, Tuple

N_VIEWS = 256


class StaticDealer:
    def __init__(self, n_items: int, world: int = 1, rank: int = 0, n_views: int = N_VIEWS):
        self._views = [(s * world + rank) % n_views for s in range(n_items)]
        self._i = 0

    def next(self) -> Optional[int]:
        if self._i >= len(self._views):
            return None
        v = self._views[self._i]
        self._i += 1
        return v


class DynamicDealer:
    """Pulls view indices 0 .. n_total-1 (mod n_views) from a counter shared by all
    ranks. ``store`` is a torch.distributed Store (or None for one process)."""

    def __init__(self, n_total: int, store=None, key: str = "nx_next_view", n_views: int = N_VIEWS, start: int = 0):
        self.n_total, self.store, self.key, self.n_views, self.start = n_total, store, key, n_views, start
        self._local = 0

    def next(self) -> Optional[int]:
        if self.store is None:
            i = self._local
            self._local += 1
        else:
            i = int(self.store.add(self.key, 1)) - 1
        if i >= self.n_total:
            return None
        return (self.start + i) % self.n_views


@dataclass
class ShardPlan:
    """View groups x image bands (config 4)."""
    world: int
    rank: int
    bands: int

    def __post_init__(self):
        if self.bands < 1 or self.world % self.bands:
            raise ValueError(f"bands ({self.bands}) must divide the world size ({self.world})")
        self.groups = self.world // self.bands
        self.group, self.band = divmod(self.rank, self.bands)

    def band_rows(self, height: int) -> Tuple[int, int]:
        from .api import image_bands
        return image_bands(height, self.bands)[self.band]

    def views(self, n_steps: int, n_views: int = N_VIEWS) -> List[int]:
        """The view this rank's group renders at each step (one per step)."""
        return [(s * self.groups + self.group) % n_views for s in range(n_steps)]


def render_dealt(renderer, dscene, cams, frames, dealer, on_frame=None) -> List[int]:
    """Renders the views the dealer hands out into the given frames (round robin, so
    len(frames) frames are in flight); returns the views rendered, in order. ``cams``
    maps a view index to its Camera. ``on_frame(view, frame)`` runs after each render
    is queued (e.g. a download)."""
    done = []
    while True:
        v = dealer.next()
        if v is None:
            return done
        f = frames[len(done) % len(frames)]
        renderer.render(dscene, cams[v], f)
        if on_frame is not None:
            on_frame(v, f)
        done.append(v)
