"""Memory-level tetrominoes: 1-D slab decomposition of axis 0 over the GPUs of
one box, with deep halos exchanged once per round of k fused steps.

This generalises the reference's two-worker deep-halo partition
(proj/src/scheduler.cpp:108-140 plan_partition, :201-435 HaloWorker,
:441-554 run_heterogeneous_impl) to P equal slabs, GPU-only (the paper's
CPU+GPU ratio split is out of scope per the north star):

* halo depth = r * k (scheduler.cpp:123), so one exchange per k-step round
  suffices; ghost rows are recomputed redundantly, the result is unchanged;
* per round each seam carries one message per direction
  (scheduler.cpp:371-406): a rank sends its first / last `depth` own planes
  and receives its neighbours' into its ghost planes;
* axis-0 planes are contiguous in both the host and the device layout, so a
  slab message is a zero-copy view of the grid buffer (no pack kernels);
* on the GPU the exchange is NCCL point-to-point (torch.distributed
  batch_isend_irecv over NVLink/NVSwitch); the same protocol runs on gloo +
  CPU tensors in the tests, with the oracle as the step engine.

* overlap (north star tier 3): each round first launches the slab's interior
  planes, whose k-step dependency cone stays inside the owned planes, while
  the exchange runs on a separate CUDA stream; the 2*depth seam planes are
  launched once the ghosts have landed (tsr_sweep_range, the reference's
  "compute interior of step 0 -> recv and install ghost -> finish seam"
  ordering of HaloWorker::run_round, scheduler.cpp:371-406).

* transport="peer" (the B200 path, north star tier 3 over NVLink): no
  message at all.  Neighbour slabs map each other's buffers with CUDA IPC;
  the seam pass of round n stores its planes both locally and straight into
  the neighbours' next-buffer ghost planes (tsr_sweep_range_mirror: the
  compute and the transfer are one kernel), then bumps a round flag in the
  neighbours' memory; before its own seam pass a rank waits on its flags
  (tsr_peer_wait).  The interior pass never waits.  See PeerLink.

Seam-side halo planes of a local slab are beyond the ghost region and never
influence owned rows; ``poison=True`` fills them with NaN to prove it (the
reference's run_heterogeneous_instrumented, scheduler.cpp:410-421).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class SlabPlan:
    """PartitionPlan (scheduler.hpp:49-64) for one rank of P equal slabs."""
    world: int
    rank: int
    global_extent: list
    halo: list
    radius: int
    fused_steps: int
    depth: int          # halo depth r*k (PartitionPlan::halo_depth)
    own_lo: int         # first owned global row (axis 0)
    own_hi: int         # one past the last owned row
    ghost_lo: int       # ghost rows below (0 on rank 0)
    ghost_hi: int       # ghost rows above (0 on the last rank)
    bytes_per_message: int = 0

    @property
    def own(self) -> int:
        return self.own_hi - self.own_lo

    @property
    def local_extent(self) -> list:
        return [self.ghost_lo + self.own + self.ghost_hi] + list(self.global_extent[1:])

    def local_row(self, global_row: int) -> int:
        return global_row - self.own_lo + self.ghost_lo


def plan_slabs(global_extent, radius: int, fused_steps: int, world: int, rank: int,
               halo=None, esize: int = 8) -> SlabPlan:
    global_extent = [int(e) for e in global_extent]
    halo = [radius] * len(global_extent) if halo is None else [int(h) for h in halo]
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if fused_steps < 1:
        raise ValueError("fused_steps must be >= 1")
    n0 = global_extent[0]
    base, extra = divmod(n0, world)
    own_lo = rank * base + min(rank, extra)
    own_hi = own_lo + base + (1 if rank < extra else 0)
    depth = radius * fused_steps
    if world > 1 and base < depth:
        raise ValueError("subdomain smaller than the halo depth")  # scheduler.cpp:454
    ghost_lo = depth if rank > 0 else 0
    ghost_hi = depth if rank < world - 1 else 0
    cross = 1
    for e in global_extent[1:]:
        cross *= e
    return SlabPlan(world, rank, global_extent, halo, radius, fused_steps, depth, own_lo,
                    own_hi, ghost_lo, ghost_hi, depth * cross * esize)


def mirror_shift(plan: SlabPlan, side: str) -> int:
    """Plane shift of a seam pass on `side` ("lo" or "hi"): my boundary own
    plane at local row j lands on the neighbour's ghost plane at local row
    j + shift (its ghost_hi planes for "lo", its ghost_lo planes for "hi")."""
    if side == "lo":
        nb = plan_slabs(plan.global_extent, plan.radius, plan.fused_steps, plan.world,
                        plan.rank - 1, plan.halo)
        return (nb.ghost_lo + nb.own) - plan.ghost_lo
    if side == "hi":
        return -(plan.ghost_lo + plan.own - plan.depth)
    raise ValueError("side must be 'lo' or 'hi'")


def local_from_global(global_grid, plan: SlabPlan, poison: bool = False):
    """Host local slab: owned rows + ghost rows (+ global halo at the true
    ends) copied from a global host grid (HaloWorker::copy_from_global,
    scheduler.cpp:236-262)."""
    h0 = plan.halo[0]
    loc = type(global_grid)(plan.local_extent, plan.halo)
    g0 = plan.own_lo - plan.ghost_lo  # global row of local row 0
    for w in (0, 1):
        src = global_grid.padded(w)
        dst = loc.padded(w)
        for lr in range(-h0, plan.local_extent[0] + h0):
            gr = g0 + lr
            seam_halo = ((lr < 0 and plan.rank > 0) or
                         (lr >= plan.local_extent[0] and plan.rank < plan.world - 1))
            if seam_halo:
                dst[lr + h0] = np.nan if poison else 0.0
            elif -h0 <= gr < global_grid.extent[0] + h0:
                dst[lr + h0] = src[gr + h0]
    if global_grid.parity:
        loc.flip_parity()
    return loc


from .scheduler import CommLog, CommRecord  # noqa: E402  (scheduler.hpp:75-88)


class _DeviceState:
    """Local slab in HBM, stepped by the engine library (tsr_advance)."""

    def __init__(self, ts, kernel, host_local, device, fused_steps, mode):
        self.ts = ts
        self.kernel = kernel
        self.dg = ts.DeviceGrid(host_local, device)
        self.fused_steps = fused_steps
        self.mode = mode
        self.h0 = host_local.halo[0]
        # element offset of local plane `row`: whole padded planes for 2-D/3-D;
        # a 1-D row is one element, its interior starts at the layout origin
        if len(host_local.extent) > 1:
            self.plane, self.base = self.dg.layout.pitch[0], self.h0 * self.dg.layout.pitch[0]
        else:
            self.plane, self.base = 1, self.dg.layout.origin

    def advance(self, n):
        return self.dg.advance(self.kernel, n, fused_steps=self.fused_steps, mode=self.mode)

    # -- overlapped rounds (tsr_sweep_range on two streams) ---------------
    def comm_stream(self):
        if not hasattr(self, "_xs"):
            torch = self.dg.torch
            self._xs = torch.cuda.Stream(device=self.dg.device)
            self._ev_ready = torch.cuda.Event()
            self._ev_comm = torch.cuda.Event()
        return self._xs

    def round_begin(self):
        """The comm stream may touch the current buffer once every launch
        that wrote it (the previous round) has finished."""
        torch = self.dg.torch
        xs = self.comm_stream()
        self._ev_ready.record(torch.cuda.current_stream(self.dg.device))
        xs.wait_event(self._ev_ready)
        return torch.cuda.stream(xs)

    def comm_done(self):
        torch = self.dg.torch
        self._ev_comm.record(self._xs)
        torch.cuda.current_stream(self.dg.device).wait_event(self._ev_comm)

    def sweep_range(self, lo, hi, n, mirror=0, mirror_planes=0):
        return self.dg.sweep_range(self.kernel, lo, hi, n, fused_steps=self.fused_steps,
                                   mode=self.mode, mirror=mirror, mirror_planes=mirror_planes)

    def flip(self, n):
        self.dg.flip(n)

    def planes(self, row: int, count: int):
        """Contiguous view of local planes [row, row+count) of the current buffer."""
        start = self.base + row * self.plane
        return self.dg.buf[self.dg.cur][start:start + count * self.plane]

    def sync(self):
        self.dg.torch.cuda.current_stream(self.dg.device).synchronize()

    def download(self, host_local):
        self.dg.download(host_local)


class _HostState:
    """Local slab on the host stepped by an injected CPU engine (tests only:
    the product never steps on the CPU)."""

    def __init__(self, host_local, step_fn):
        import torch
        self.torch = torch
        self.g = host_local
        self.step_fn = step_fn
        self.h0 = host_local.halo[0]
        self.plane = host_local.stride(0) if host_local.dims > 1 else 1

    def advance(self, n):
        self.step_fn(self.g, n)

        class _S:
            kernel_launches = 0
        return _S()

    def planes(self, row: int, count: int):
        start = (row + self.h0) * self.plane
        return self.torch.from_numpy(self.g.read_data()[start:start + count * self.plane])

    def sync(self):
        pass

    # overlapped rounds on the host: the same range / flip protocol, one
    # pass of n steps per range computed on a scratch copy
    def round_begin(self):
        import contextlib
        return contextlib.nullcontext()

    def comm_done(self):
        pass

    def sweep_range(self, lo, hi, n):
        if hi <= lo:
            return 0
        tmp = self.g.copy()
        self.step_fn(tmp, n)
        h = self.h0
        self.g.padded(1 - self.g.parity)[lo + h:hi + h] = tmp.padded(tmp.parity)[lo + h:hi + h]
        return 0

    def flip(self, n):
        self.g.flip_parity()


class PeerLink:
    """CUDA-IPC mappings of the neighbour slabs' two buffers and round flags
    (csrc/peer.cu).  Collective constructor: every rank of `group` calls it.

    flags[0] / flags[1] of a rank count the rounds its lo / hi neighbour has
    completed; a rank signals round completion into its lo neighbour's
    flags[1] and its hi neighbour's flags[0]."""

    def __init__(self, plan: SlabPlan, dg, group=None):
        import torch
        import torch.distributed as dist
        from . import _abi
        self._abi = _abi
        self.dist, self.group = dist, group
        self.torch = torch
        self.dg = dg
        # [rounds the lo neighbour completed, ... the hi neighbour, rounds I completed]
        self.flags = torch.zeros(3, dtype=torch.int32, device=dg.device)
        torch.cuda.synchronize(dg.device)
        mine = {"rank": plan.rank, "buf": [_abi.ipc_export(dg.ptr(0)), _abi.ipc_export(dg.ptr(1))],
                "flags": _abi.ipc_export(self.flags.data_ptr())}
        info = [None] * plan.world
        dist.all_gather_object(info, mine, group=group)
        self._bases = {}
        self.peer = {}
        err = None
        try:
            for side, nb in (("lo", plan.rank - 1), ("hi", plan.rank + 1)):
                if not 0 <= nb < plan.world:
                    continue
                peer = info[nb]
                shift = mirror_shift(plan, side)
                word = 1 if side == "lo" else 0  # the flag word of mine it counts in
                self.peer[side] = {"buf": [self._map(*peer["buf"][0]),
                                           self._map(*peer["buf"][1])],
                                   "flag": self._map(*peer["flags"]) + 4 * word,
                                   "shift": shift}
        except Exception as e:  # noqa: BLE001 - reported collectively below
            err = f"rank {plan.rank}: {e}"
        errs = [None] * plan.world
        dist.all_gather_object(errs, err, group=group)
        failed = [e for e in errs if e]
        if failed:  # every rank gives up together (no rank left waiting on a flag)
            for base in self._bases.values():
                self._abi.ipc_close(base)
            self._bases, self.peer = {}, {}
            raise RuntimeError("peer mapping failed: " + "; ".join(failed))
        dist.barrier(group=group)

    def _map(self, handle: bytes, offset: int) -> int:
        if handle not in self._bases:
            self._bases[handle] = self._abi.ipc_open(handle)
        return self._bases[handle] + offset

    def _stream(self) -> int:
        return self.torch.cuda.current_stream(self.dg.device).cuda_stream

    def wait(self) -> int:
        """Later work on the current stream waits until both neighbours have
        completed as many rounds as this rank (the device-side counter), so
        the call has no per-round arguments and can sit in a CUDA graph.
        Returns the kernels launched."""
        f = self.flags.data_ptr()
        lo = f if "lo" in self.peer else None
        hi = f + 4 if "hi" in self.peer else None
        self._abi.check(self._abi.lib().tsr_peer_round_wait(lo, hi, f + 8, self._stream()))
        return 1

    def signal(self) -> int:
        """Counts this rank's round and publishes the count to both
        neighbours (after all earlier work on the stream)."""
        lo = self.peer["lo"]["flag"] if "lo" in self.peer else None
        hi = self.peer["hi"]["flag"] if "hi" in self.peer else None
        self._abi.check(self._abi.lib().tsr_peer_round_signal(lo, hi, self.flags.data_ptr() + 8,
                                                              self._stream()))
        return 1

    def mirror(self, side: str, which: int) -> tuple[int, int]:
        """(address of the neighbour's buffer `which`, plane shift) for a seam
        pass on `side`."""
        p = self.peer[side]
        return p["buf"][which], p["shift"]

    def close(self) -> None:
        """Collective: no rank unmaps before every rank's stores have landed."""
        self.torch.cuda.synchronize(self.dg.device)
        self.dist.barrier(group=self.group)
        for base in self._bases.values():
            self._abi.ipc_close(base)
        self._bases = {}
        self.peer = {}


class SlabRunner:
    """Round driver for one rank (HaloWorker::run_round generalised to P
    slabs).  ``advance(n)`` runs one round of n <= k steps: exchange the
    ghost planes with both neighbours, then n fused steps on the local slab."""

    def __init__(self, plan: SlabPlan, state, group=None, overlap: bool = True,
                 transport: str = "nccl", graphs: bool = False):
        import torch.distributed as dist
        if transport not in ("nccl", "peer"):
            raise ValueError("transport must be 'nccl' or 'peer'")
        self.dist = dist
        # gloo cannot move CUDA tensors point-to-point: stage through host
        # memory (tests run several ranks on one GPU this way); NCCL sends
        # straight from HBM.
        self.stage_via_host = (dist.is_initialized() and
                               dist.get_backend(group) == "gloo")
        self.plan = plan
        self.state = state
        self.group = group
        self.fused_steps = plan.fused_steps
        self.overlap = overlap
        self.round = 0
        self.log = CommLog()
        self.exchange_bytes = 0
        self.transport = transport
        self.link = None
        # peer transport: after the first full round, one CUDA graph per
        # buffer parity is recorded and every later full round replays one
        self.graphs = graphs
        self._graph = {}
        self.graphs_captured = 0
        if transport == "peer" and plan.world > 1:
            if not isinstance(state, _DeviceState):
                raise ValueError("the peer transport needs device slabs")
            # ghosts consistent before the first round (one message exchange,
            # outside any timed region), then IPC mappings for the rounds
            self.exchange()
            self.link = PeerLink(plan, state.dg, group)

    # -- constructors -----------------------------------------------------
    @classmethod
    def on_device(cls, ts, kernel, plan: SlabPlan, host_local, device, mode="exact",
                  group=None, overlap=True, transport="nccl", graphs=False):
        return cls(plan, _DeviceState(ts, kernel, host_local, device, plan.fused_steps, mode),
                   group, overlap, transport, graphs)

    @classmethod
    def synthetic(cls, ts, kernel, plan: SlabPlan, dtype, device, seed=1, fused_steps=None,
                  mode="exact", group=None, overlap=True, transport="nccl", graphs=False):
        """Benchmark slab: the local grid gets the GLOBAL grid's
        fill_random(seed) values for its rows (the mt19937_64 stream advanced
        past the rows below it), without building the global host grid; the
        ghost rows match the neighbours' from the start."""
        from . import _abi
        cls_ = ts.Grid if dtype == "f64" else ts.GridF
        # resolve the engine's k on the local geometry
        desc = _abi.grid_desc(plan.local_extent, plan.halo, dtype)
        _, k = _abi.query_plan(kernel, desc, fused_steps or 0, mode)
        if k != plan.fused_steps:
            esize = 8 if dtype == "f64" else 4
            plan = plan_slabs(plan.global_extent, plan.radius, k, plan.world, plan.rank,
                              plan.halo, esize)
        host = cls_(plan.local_extent, plan.halo)
        cross = 1
        for e in plan.global_extent[1:]:
            cross *= e
        ts.fill_random(host, seed, skip=(plan.own_lo - plan.ghost_lo) * cross)
        return cls.on_device(ts, kernel, plan, host, device, mode, group, overlap, transport,
                             graphs)

    @classmethod
    def on_host(cls, plan: SlabPlan, host_local, step_fn, group=None, overlap=False):
        return cls(plan, _HostState(host_local, step_fn), group, overlap)

    # -- protocol ---------------------------------------------------------
    def exchange(self):
        """One message per direction per seam (scheduler.cpp:371-381)."""
        p, dist = self.plan, self.dist
        d = p.depth
        sends, recvs = [], []  # (peer, tensor)
        if p.rank > 0:
            sends.append((p.rank - 1, self.state.planes(p.ghost_lo, d)))
            recvs.append((p.rank - 1, self.state.planes(0, d)))
            self.log.records.append(CommRecord(self.round, f"r{p.rank - 1}_to_r{p.rank}",
                                               p.bytes_per_message))
        if p.rank < p.world - 1:
            sends.append((p.rank + 1, self.state.planes(p.ghost_lo + p.own - d, d)))
            recvs.append((p.rank + 1, self.state.planes(p.ghost_lo + p.own, d)))
            self.log.records.append(CommRecord(self.round, f"r{p.rank + 1}_to_r{p.rank}",
                                               p.bytes_per_message))
        if not sends:
            return
        staged = None
        if self.stage_via_host and sends[0][1].is_cuda:
            self.state.sync()
            sends = [(peer, t.cpu()) for peer, t in sends]
            staged = recvs
            recvs = [(peer, t.new_empty(t.shape, device="cpu")) for peer, t in recvs]
        ops = [dist.P2POp(dist.isend, t, peer, self.group) for peer, t in sends]
        ops += [dist.P2POp(dist.irecv, t, peer, self.group) for peer, t in recvs]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if staged is not None:
            for (peer, dst), (_, src) in zip(staged, recvs):
                dst.copy_(src)
        for _, t in sends:
            self.exchange_bytes += t.numel() * t.element_size()

    def ranges(self, n: int, depth: int = 0):
        """(interior, seams) plane ranges of one overlapped round in local
        interior coordinates: the interior's n-step cone stays inside the
        owned planes; the seams need the ghosts.  `depth` widens the seams
        to that many planes (the peer transport's seams are the planes the
        neighbours' ghosts receive: always the full r*k)."""
        p = self.plan
        d = max(p.radius * n, depth)
        dl = d if p.ghost_lo else 0
        dh = d if p.ghost_hi else 0
        lo, hi = p.ghost_lo, p.ghost_lo + p.own
        if hi - lo <= dl + dh:
            return (lo, lo), [(lo, hi)]
        return (lo + dl, hi - dh), [(lo, lo + dl), (hi - dh, hi)]

    def _peer_launches(self, n: int) -> int:
        """The GPU work of one peer round (no host-side state changes, so it
        can be captured): interior pass, wait, seam passes into the
        neighbours' ghost planes, signal."""
        st, link, p = self.state, self.link, self.plan
        (ilo, ihi), seams = self.ranges(n, depth=p.depth)
        launches = st.sweep_range(ilo, ihi, n)
        launches += link.wait()
        nxt = 1 - st.dg.cur
        first, last = p.ghost_lo, p.ghost_lo + p.own
        # the depth planes each neighbour's ghosts receive
        mirrored = []
        if "lo" in link.peer:
            mirrored.append(("lo", first, min(last, first + p.depth)))
        if "hi" in link.peer:
            mirrored.append(("hi", max(first, last - p.depth), last))
        # seam planes no mirrored pass covers (only in a slab thinner than 2
        # seams plus the interior cone): plain passes
        for lo, hi in seams:
            for _, a, b in mirrored:
                if a <= lo < b:
                    lo = b
                if a < hi <= b:
                    hi = a
            if hi > lo:
                launches += st.sweep_range(lo, hi, n)
        for side, a, b in mirrored:
            addr, shift = link.mirror(side, nxt)
            launches += st.sweep_range(a, b, n, mirror=addr, mirror_planes=shift)
        launches += link.signal()
        return launches

    def _capture(self, cur: int, n: int) -> None:
        """Records the launches of a full peer round whose current buffer is
        `cur` into a CUDA graph (recording executes nothing; the buffer
        index is set for the recording and restored)."""
        import torch
        dg = self.state.dg
        keep = dg.cur
        dg.cur = cur
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                launches = self._peer_launches(n)
        finally:
            dg.cur = keep
        self._graph[(cur, n)] = (g, launches)
        self.graphs_captured += 1

    def _round_peer(self, n: int):
        """One round over peer memory: eager the first time (kernels load),
        then — with graphs — both buffer parities are recorded once and
        every later full round is one graph replay."""
        st, p = self.state, self.plan
        key = (st.dg.cur, n)
        if self.graphs and key in self._graph:
            g, launches = self._graph[key]
            g.replay()
        else:
            launches = self._peer_launches(n)
            if self.graphs and n == self.fused_steps:
                for cur in (0, 1):
                    if (cur, n) not in self._graph:
                        self._capture(cur, n)
        for side in ("lo", "hi"):
            if side in self.link.peer:
                self.exchange_bytes += p.bytes_per_message
                self.log.records.append(CommRecord(self.round, f"r{p.rank}_to_{side}",
                                                   p.bytes_per_message))
        st.flip(n)

        class _S:
            kernel_launches = launches
        return _S()

    def _round_overlapped(self, n: int):
        """HaloWorker::run_round's order (scheduler.cpp:371-406) on two
        streams: exchange on the comm stream || interior planes on the
        compute stream, then the seam planes once the ghosts are in."""
        st = self.state
        with st.round_begin():
            self.exchange()
        (ilo, ihi), seams = self.ranges(n)
        launches = st.sweep_range(ilo, ihi, n)
        st.comm_done()
        for lo, hi in seams:
            launches += st.sweep_range(lo, hi, n)
        st.flip(n)

        class _S:
            kernel_launches = launches
        return _S()

    def advance(self, n: int):
        if n > self.fused_steps:
            raise ValueError("a round advances at most k = depth / r steps")
        if self.link is not None:
            st = self._round_peer(n)
        elif self.plan.world > 1 and self.overlap:
            st = self._round_overlapped(n)
        else:
            if self.plan.world > 1:
                self.exchange()
            st = self.state.advance(n)
        # ghost planes recomputed by this rank (HaloWorker::tally_ghost)
        cross = 1
        for e in self.plan.global_extent[1:]:
            cross *= e
        self.log.ghost_recompute_points += (self.plan.ghost_lo + self.plan.ghost_hi) * cross * n
        self.round += 1
        return st

    def run(self, steps: int):
        """ceil(T/k) rounds (scheduler.cpp:471-474)."""
        left = int(steps)
        while left > 0:
            n = min(self.fused_steps, left)
            self.advance(n)
            left -= n

    def own_rows(self, host_local=None):
        """Owned rows of the local read buffer as a padded-shape ndarray (a
        device state is first downloaded into `host_local`)."""
        if host_local is not None:
            self.state.download(host_local)
            g = host_local
        else:
            g = self.state.g
        h0 = g.halo[0]
        return g.padded(g.parity)[h0 + self.plan.ghost_lo:h0 + self.plan.ghost_lo + self.plan.own]

    def close(self) -> None:
        """Collective teardown of the peer mappings (no-op for NCCL)."""
        self._graph = {}
        if self.link is not None:
            self.link.close()
            self.link = None

    def comm_summary(self) -> dict:
        return {"rounds": self.round, "transport": self.transport if self.plan.world > 1 else None,
                "graphs_captured": self.graphs_captured,
                "overlap": bool(self.overlap and self.plan.world > 1),
                "messages_sent": len(self.log.records),
                "bytes_per_message": self.plan.bytes_per_message,
                "halo_depth": self.plan.depth, "fused_steps": self.fused_steps,
                "bytes_sent": self.exchange_bytes,
                "ghost_recompute_points": self.log.ghost_recompute_points}
