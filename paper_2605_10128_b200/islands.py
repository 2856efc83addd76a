"""Island MapElites across GPUs (BASELINE.json north_star):
one process per GPU, each running its own population and archive on the
device; every `merge_every` generations the archives are exchanged with one
NCCL allgather of fixed-size archive blobs and merged on the device.

The reference runs a single population (run_optimizer,
/root/reference/proj/src/qd_optimizer.cpp:344-417); island mode is the
north_star's multi-GPU form. The merge keeps the reference's archive
semantics: it re-inserts every island's entries in (island, cell, position)
order with Repertoire::insert (qd_optimizer.cpp:281-303: non-finite fitness
rejected, duplicate canonical key in the cell rejected, a full cell only takes
a strictly better entry, ties go after existing entries). Every island that
merges the same gathered blobs therefore holds the same archive, and a run
with one island is unchanged by a merge.

Blob layout (mirrors tgb::BlobLayout in csrc/cuda/qd.cuh; S = cells x cap
slots, cell-major, position-minor; all sections 8-byte aligned):
fitness, lambda_o, lambda_b f64[S]; worst_energy f64[S*worst_k];
genome i32[S*n_slots]; lambda_c, lambda_c0, lambda_d, lambda_s, lambda_r,
worst_n i32[S]; worst_idx i32[S*worst_k]. Empty slots carry fitness -inf.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

_F64 = ("fitness", "lambda_o", "lambda_b")
_I32 = ("lambda_c", "lambda_c0", "lambda_d", "lambda_s", "lambda_r", "worst_n")


def _al(x: int) -> int:
    return (x + 7) & ~7


@dataclass(frozen=True)
class BlobLayout:
    cells: int
    cap: int
    n_slots: int
    worst_k: int

    @property
    def slots(self) -> int:
        return self.cells * self.cap

    def offsets(self) -> Dict[str, int]:
        S, ns, wk = self.slots, self.n_slots, self.worst_k
        o, out = 0, {}
        for name, nbytes in (("fitness", S * 8), ("lambda_o", S * 8), ("lambda_b", S * 8),
                             ("worst_energy", S * wk * 8), ("genome", S * ns * 4), ("lambda_c", S * 4),
                             ("lambda_c0", S * 4), ("lambda_d", S * 4), ("lambda_s", S * 4), ("lambda_r", S * 4),
                             ("worst_n", S * 4), ("worst_idx", S * wk * 4)):
            out[name] = o
            o += _al(nbytes)
        out["total"] = o
        return out

    @property
    def nbytes(self) -> int:
        return self.offsets()["total"]

    def views(self, buf: np.ndarray) -> Dict[str, np.ndarray]:
        """Typed numpy views of one blob (uint8 array of nbytes)."""
        off = self.offsets()
        S, ns, wk = self.slots, self.n_slots, self.worst_k
        b = buf.view(np.uint8)
        v = {}
        for name in _F64:
            v[name] = b[off[name]:off[name] + S * 8].view(np.float64)
        v["worst_energy"] = b[off["worst_energy"]:off["worst_energy"] + S * wk * 8].view(np.float64).reshape(S, wk)
        v["genome"] = b[off["genome"]:off["genome"] + S * ns * 4].view(np.int32).reshape(S, ns)
        for name in _I32:
            v[name] = b[off[name]:off[name] + S * 4].view(np.int32)
        v["worst_idx"] = b[off["worst_idx"]:off["worst_idx"] + S * wk * 4].view(np.int32).reshape(S, wk)
        return v


def pack_entries(layout: BlobLayout, entries: Sequence) -> np.ndarray:
    """Host encoder of an archive snapshot (RepertoireSnapshot.entries, cell
    order, position order inside a cell) into one island blob, e.g. to seed an
    island from a saved snapshot."""
    buf = np.zeros(layout.nbytes, np.uint8)
    v = layout.views(buf)
    v["fitness"][:] = -np.inf
    v["genome"][:] = -1
    fill: Dict[int, int] = {}
    for e in entries:
        pos = fill.get(e.cell, 0)
        if pos >= layout.cap:
            raise ValueError(f"cell {e.cell} holds more than {layout.cap} entries")
        fill[e.cell] = pos + 1
        i = e.cell * layout.cap + pos
        s = e.score
        v["genome"][i] = list(e.genome.action_slots) + list(e.genome.disconnection_slots)
        v["fitness"][i] = s.fitness
        v["lambda_o"][i] = s.lambda_o
        v["lambda_b"][i] = s.lambda_b
        for name in _I32[:-1]:
            v[name][i] = getattr(s, name)
        wl = list(s.worst_contingencies)[:layout.worst_k]
        v["worst_n"][i] = len(wl)
        for j, (k, en) in enumerate(wl):
            v["worst_idx"][i, j] = k
            v["worst_energy"][i, j] = en
    return buf


def unpack_blob(layout: BlobLayout, buf: np.ndarray) -> List[dict]:
    """Live entries of one blob in (cell, position) order."""
    v = layout.views(np.ascontiguousarray(buf))
    out = []
    for i in range(layout.slots):
        f = float(v["fitness"][i])
        if not np.isfinite(f):
            continue
        wn = int(v["worst_n"][i])
        out.append({"cell": i // layout.cap, "genome": v["genome"][i].tolist(), "fitness": f,
                    "lambda_o": float(v["lambda_o"][i]), "lambda_b": float(v["lambda_b"][i]),
                    **{name: int(v[name][i]) for name in _I32[:-1]},
                    "worst": [(int(v["worst_idx"][i, j]), float(v["worst_energy"][i, j])) for j in range(wn)]})
    return out


class IslandExchange:
    """Allgather + device merge of the archives of all ranks of `group`.

    The blobs never leave device memory: pack (kernel) -> NCCL allgather ->
    merge (kernels), all ordered on the engine context's stream."""

    def __init__(self, session, group=None):
        import torch
        import torch.distributed as dist

        from . import api

        self.session = session
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        # NCCL gathers device buffers directly; any other backend (gloo: the
        # single-GPU test harness of the N>1 path) is staged through host memory
        self.device_collective = not dist.is_initialized() or dist.get_backend(group) == "nccl"
        self.nbytes = session.blob_bytes()
        dev = torch.device("cuda", torch.cuda.current_device())
        self.send = torch.empty(self.nbytes, dtype=torch.uint8, device=dev)
        self.recv = torch.empty(self.nbytes * self.world, dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.ExternalStream(api.context_stream(session.ctx), device=dev)
        self.exchanges = 0

    def exchange(self) -> None:
        import torch
        import torch.distributed as dist

        with torch.cuda.stream(self.stream):
            self.session.pack(self.send.data_ptr())
            if self.world == 1:
                self.session.merge(self.send.data_ptr(), 1)
            elif self.device_collective:
                dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
                self.session.merge(self.recv.data_ptr(), self.world)
            else:
                host = self.send.cpu()
                gathered = torch.empty(self.world * self.nbytes, dtype=torch.uint8)
                dist.all_gather_into_tensor(gathered, host, group=self.group)
                self.recv.copy_(gathered)
                self.session.merge(self.recv.data_ptr(), self.world)
        self.exchanges += 1


class BatchShard:
    """Batch-sharded generations (SURVEY.md 8(e) parity mode): the ranks of
    `group` share ONE population. Every rank draws the same offspring (lane
    seeds depend only on (seed, iteration, lane), qd_optimizer.cpp:377-383),
    evaluates its slice of lanes, the score slices are allgathered (NCCL, device
    blobs) and every rank inserts all lanes in lane order: the archive is
    bit-identical to a one-GPU run (strong scaling of one generation)."""

    def __init__(self, session, group=None):
        import torch
        import torch.distributed as dist

        from . import api

        self.session = session
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        B = session.cfg.batch_size
        if B % self.world:
            raise api.ConfigError(f"batch {B} does not split evenly over {self.world} ranks")
        self.per = B // self.world
        self.lo, self.hi = self.rank * self.per, (self.rank + 1) * self.per
        self.nbytes = session.scores_blob_bytes(self.per)
        self.device_collective = not dist.is_initialized() or dist.get_backend(group) == "nccl"
        dev = torch.device("cuda", torch.cuda.current_device())
        self.send = torch.empty(self.nbytes, dtype=torch.uint8, device=dev)
        self.recv = torch.empty(self.nbytes * self.world, dtype=torch.uint8, device=dev)
        self.stream = torch.cuda.ExternalStream(api.context_stream(session.ctx), device=dev)

    def step(self, n: int = 1) -> None:
        import torch
        import torch.distributed as dist

        s = self.session
        with torch.cuda.stream(self.stream):
            for _ in range(n):
                s.generation_begin()
                s.evaluate_lanes(self.lo, self.hi)
                if self.world > 1:
                    s.scores_pack(self.lo, self.hi, self.send.data_ptr())
                    if self.device_collective:
                        dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
                    else:
                        gathered = torch.empty(self.world * self.nbytes, dtype=torch.uint8)
                        dist.all_gather_into_tensor(gathered, self.send.cpu(), group=self.group)
                        self.recv.copy_(gathered)
                    for r in range(self.world):
                        if r != self.rank:
                            s.scores_unpack(r * self.per, (r + 1) * self.per, self.recv[r * self.nbytes:].data_ptr())
                s.generation_end()


class NativeIslands:
    """The same two exchanges through the engine's own NCCL communicator
    (tg_islands_*, host/islands.cpp): ncclAllGather on the context stream
    between the pack / merge (island mode) or score pack / unpack (shard mode)
    kernels; no torch on the data path. torch.distributed only carries the
    128-byte NCCL unique id from rank 0 to the others (any backend)."""

    def __init__(self, session, group=None):
        import ctypes as C

        import numpy as np
        import torch
        import torch.distributed as dist

        from . import api

        self.session = session
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = np.zeros(128, np.uint8)
        if self.rank == 0:
            api._check(api.LIB.tg_islands_unique_id(uid.ctypes.data_as(C.c_void_p)))
        if self.world > 1:
            t = torch.from_numpy(uid)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            uid = t.cpu().numpy().astype(np.uint8)
        h = C.c_void_p()
        api._check(api.LIB.tg_islands_create(session.ctx._h, uid.ctypes.data_as(C.c_void_p), self.rank, self.world,
                                             C.byref(h)))
        self._h = h
        self.exchanges = 0

    def exchange(self) -> None:
        from . import api

        api._check(api.LIB.tg_islands_exchange(self._h))
        self.exchanges += 1

    def step(self, n: int = 1, merge_every: int = 1) -> None:
        """n island generations, an exchange after every merge_every-th (0 = none)."""
        from . import api

        api._check(api.LIB.tg_islands_step(self._h, n, merge_every))
        if merge_every:
            self.exchanges += n // merge_every

    def shard_step(self, n: int = 1) -> None:
        """n batch-sharded generations of one population (BatchShard semantics)."""
        from . import api

        api._check(api.LIB.tg_islands_shard_step(self._h, n, self.session.cfg.batch_size))

    def __del__(self):
        from . import api

        if getattr(self, "_h", None):
            api.LIB.tg_islands_destroy(self._h)
            self._h = None


def run_islands(session, generations: int, merge_every: int = 1, exchange: Optional[IslandExchange] = None) -> None:
    """`generations` MapElites generations of this island with an archive
    merge every `merge_every` generations (0 = never)."""
    ex = exchange
    if merge_every and ex is None:
        ex = IslandExchange(session)
    done = 0
    while done < generations:
        n = generations - done if not merge_every else min(merge_every, generations - done)
        session.step(n)
        done += n
        if merge_every and done % merge_every == 0:
            ex.exchange()
