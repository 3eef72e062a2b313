"""Collective contract of the grid and its two executors.

Reference contract (/root/reference/pkg/src/gridlp/comm.py): axis-scoped
sum-AllReduce — R reduces down a grid column (over i), C along a grid row
(over j), G over all devices — with deterministic ascending-rank order
(:75-84), replicated results and per-device logical counters that count
every call, even on singleton groups (:322-335).

Executors:
  * `VirtualGrid` — one process, one GPU, every block of the R x C grid
    resident in that GPU's HBM. A vector reduction is the ascending-order
    sum of the block partials, fused into the consuming epilogue kernel
    (bit-identical to the reference's simulated grid).
  * `NcclGrid` — one process per GPU (torchrun), device (i, j) = rank
    i*C + j, NCCL over NVLink on per-column (R axis) and per-row (C axis)
    sub-communicators for the vector sums. Scalars of a pass are gathered
    once over the world group and reduced on every rank in ascending order,
    so every rank takes identical restart/termination decisions (the
    reference's "replicated, never broadcast" rule, pdhg_engine.py:18-19).
"""

from __future__ import annotations

import datetime
from collections import Counter

import numpy as np
import torch

AXES = ("R", "C", "G")


class CollectiveError(RuntimeError):
    """comm.py:45 of the reference."""


class CollectiveTimeout(CollectiveError):
    """A collective did not complete within collective_timeout_seconds
    (reference comm.py:49, :125-132)."""


class CollectiveMismatch(CollectiveError):
    """Devices issued different collective sequences (reference comm.py:53,
    the lockstep check :87-91, :309-320)."""


class WorkerError(RuntimeError):
    """A device worker raised; the original exception is chained
    (reference comm.py:57, :219-221)."""


class Ledger:
    """Logical collective counters (comm.py:61-72, :322-335). Every device
    issues the same sequence, so events are recorded once and expanded per
    device with that device's vector lengths (m_i for C, n_j for R)."""

    def __init__(self):
        self.events = Counter()   # (axis, kind, length_key) -> calls

    def vec(self, axis: str, length_key: str, times: int = 1):
        self.events[(axis, "vec", length_key)] += times

    def scalar(self, axis: str, times: int = 1):
        self.events[(axis, "scalar", "1")] += times

    def snapshot(self):
        return Counter(self.events)

    @staticmethod
    def expand(events, layout) -> list:
        R, C = layout.topology.rows, layout.topology.cols
        out = []
        for i in range(R):
            m_i = int(layout.row_cuts[i + 1] - layout.row_cuts[i])
            for j in range(C):
                n_j = int(layout.col_cuts[j + 1] - layout.col_cuts[j])
                size = {"m": m_i, "n": n_j, "1": 1}
                axes = {a: {"vector_calls": 0, "scalar_calls": 0, "elements_reduced": 0} for a in AXES}
                for (axis, kind, key), cnt in events.items():
                    d = axes[axis]
                    d["vector_calls" if kind == "vec" else "scalar_calls"] += cnt
                    d["elements_reduced"] += cnt * size[key]
                out.append({"device": [i, j], "axes": axes})
        return out

    @staticmethod
    def diff(after, before):
        d = Counter(after)
        d.subtract(before)
        return d

    @staticmethod
    def grid_total(per_device: list) -> dict:
        tot = {a: {"vector_calls": 0, "scalar_calls": 0, "elements_reduced": 0} for a in AXES}
        for entry in per_device:
            for a in AXES:
                for k in tot[a]:
                    tot[a][k] += entry["axes"][a][k]
        return tot


def asc_sum(values):
    """Ascending-order scalar reduction (comm.py:75-84)."""
    acc = values[0]
    for v in values[1:]:
        acc = acc + v
    return acc


class VirtualGrid:
    """All blocks in one process on one device."""

    kind = "virtual"

    def __init__(self, rows: int, cols: int):
        self.rows, self.cols = rows, cols
        self.local = [(i, j) for i in range(rows) for j in range(cols)]
        self.rank = 0
        self.world = 1
        self.active = True

    def reduce(self, axis, index, partials, scratch=None):
        """Return the partial list (ascending); the consuming kernel sums it."""
        return list(partials)

    def table(self, local_rows: dict) -> dict:
        return local_rows

    def gather_vectors(self, local: dict, lengths: dict, device) -> dict:
        return local

    def barrier(self):
        pass


class NcclGrid:
    """One device per rank over torch.distributed (NCCL on GPUs; gloo works
    for the host-logic tests on CPU)."""

    kind = "nccl"

    def __init__(self, rows: int, cols: int, device, timeout: float = 120.0):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise RuntimeError("NcclGrid needs an initialised torch.distributed process group")
        self.dist = dist
        self.timeout = float(timeout)
        self._td = datetime.timedelta(seconds=self.timeout)
        self._seq = 0                  # host collectives issued (lockstep tag)
        self.rows, self.cols = rows, cols
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        if self.world < rows * cols:
            raise ValueError(f"grid {rows}x{cols} needs {rows * cols} ranks, world size is {self.world}")
        self.device = device
        self.active = self.rank < rows * cols
        self.coord = (self.rank // cols, self.rank % cols) if self.active else None
        self.local = [self.coord] if self.active else []
        # every rank must create every group, in the same order; the groups'
        # own timeout bounds the device-side vector collectives (NCCL watchdog)
        td = self._td
        self.col_groups = [dist.new_group([i * cols + j for i in range(rows)], timeout=td) for j in range(cols)]
        self.row_groups = [dist.new_group([i * cols + j for j in range(cols)], timeout=td) for i in range(rows)]
        self.active_group = dist.new_group(list(range(rows * cols)), timeout=td)
        # NCCL collectives can be captured in CUDA graphs; gloo (ranks sharing
        # a GPU in tests, CPU runs) cannot
        self.graph_safe = dist.get_backend() == "nccl"

    def _wait(self, work, what: str):
        """Host-side wait on a collective, bounded by collective_timeout_seconds:
        a rank that died or stopped issuing collectives surfaces here as the
        reference's CollectiveTimeout instead of a hang."""
        try:
            ok = work.wait(timeout=self._td)
        except Exception as exc:   # torch raises on timeout / a failed peer
            raise CollectiveTimeout(f"collective {what} timed out after {self.timeout}s or failed on a peer: "
                                    f"{exc}") from exc
        if ok is False:
            raise CollectiveTimeout(f"collective {what} timed out after {self.timeout}s")

    def reduce(self, axis, index, partials, scratch=None):
        """Axis sum of the members' partial vectors in ASCENDING member order
        (the reference's order, comm.py:75-84): all-gather the partials, then
        add them in order on every member — so every rank holds the same bits
        as the virtual grid, whatever algorithm / protocol NCCL would pick
        for an allreduce (NCCL_ALGO / NCCL_PROTO do not matter). Used by the
        KKT pass and the power iteration; the main loop uses the sharded
        exchange (exchange / gather_shard), which has the same property."""
        (p,) = partials
        buf = p if scratch is None else scratch
        group = self._axis_group(axis, index)
        G = self.rows if axis == "R" else self.cols
        if G > 1:
            n = p.numel()
            stack = torch.empty((G, n), dtype=p.dtype, device=p.device)
            if self._gloo_cuda(group, p) or self.dist.get_backend(group) != "nccl":
                outs = list(stack.unbind(0))
                self.dist.all_gather(outs, p.contiguous(), group=group)
            else:
                self.dist.all_gather_into_tensor(stack.view(-1), p.contiguous(), group=group)
            buf.copy_(stack[0])
            for q in range(1, G):
                buf.add_(stack[q])
        elif scratch is not None:
            buf.copy_(p)
        return [buf]

    def _axis_group(self, axis, index):
        return self.col_groups[index] if axis == "R" else self.row_groups[index]

    def _gloo_cuda(self, group, t) -> bool:
        return t.is_cuda and self.dist.get_backend(group) == "gloo"

    def exchange(self, axis, index, partial, recv):
        """Ordered reduce-scatter, first half: recv[q*S:(q+1)*S] = member q's
        partial of this rank's shard (all-to-all over the axis group; the
        consuming epilogue adds the slices in ascending q)."""
        group = self._axis_group(axis, index)
        if self._gloo_cuda(group, partial):
            # gloo has no all-to-all on CUDA tensors (ranks sharing one GPU in
            # tests): all-gather the full partials and keep this rank's shard
            G = self.rows if axis == "R" else self.cols
            me = self.coord[0] if axis == "R" else self.coord[1]
            S = partial.numel() // G
            outs = [torch.empty_like(partial) for _ in range(G)]
            self.dist.all_gather(outs, partial, group=group)
            for q in range(G):
                recv[q * S:(q + 1) * S].copy_(outs[q][me * S:(me + 1) * S])
            return
        self.dist.all_to_all_single(recv, partial, group=group)

    def gather_shard(self, axis, index, vec, me, S):
        """All-gather this rank's shard [me*S, (me+1)*S) of `vec` (a view of
        storage padded to G*S) into every member's copy, in place."""
        group = self._axis_group(axis, index)
        G = self.rows if axis == "R" else self.cols
        if vec.storage_offset() != 0 or vec.untyped_storage().nbytes() < G * S * vec.element_size():
            raise ValueError("gather_shard needs a view at the start of storage padded to G*S elements")
        full = torch.as_strided(vec, (G * S,), (1,))      # the padded storage behind the view
        mine = full[me * S:(me + 1) * S]
        if self._gloo_cuda(group, full):
            outs = [torch.empty_like(mine) for _ in range(G)]
            self.dist.all_gather(outs, mine.contiguous(), group=group)
            for q in range(G):
                if q != me:
                    full[q * S:(q + 1) * S].copy_(outs[q])
            return
        self.dist.all_gather_into_tensor(full, mine, group=group)

    def table(self, local_rows: dict) -> dict:
        """All-gather each active rank's scalar row over the active group.
        Each row carries this rank's host-collective sequence number and row
        width; ranks that disagree issued different collective sequences
        (CollectiveMismatch, the reference's lockstep check)."""
        (coord, row), = local_rows.items()
        row = np.asarray(row, dtype=np.float64)
        self._seq += 1
        tagged = np.concatenate([[float(self._seq), float(len(row))], row])
        t = torch.as_tensor(tagged, device=self.device)
        outs = [torch.empty_like(t) for _ in range(self.rows * self.cols)]
        self._wait(self.dist.all_gather(outs, t, group=self.active_group, async_op=True), f"table#{self._seq}")
        full = torch.stack(outs).cpu().numpy()
        if not (np.all(full[:, 0] == full[0, 0]) and np.all(full[:, 1] == full[0, 1])):
            raise CollectiveMismatch(f"collective sequences diverged: (seq, width) per rank "
                                     f"{[(int(a), int(b)) for a, b in full[:, :2]]}")
        return {(r // self.cols, r % self.cols): full[r, 2:] for r in range(self.rows * self.cols)}

    def agree(self, value: str, what: str) -> None:
        """Raise RuntimeError when ranks hold different values of a replicated
        decision (solver_driver.py:242-244: diverged device statuses)."""
        got = [None] * (self.rows * self.cols)
        self.dist.all_gather_object(got, value, group=self.active_group)
        if len(set(got)) != 1:
            raise RuntimeError(f"device {what} diverged: {set(got)}")

    def gather_vectors(self, local: dict, lengths: dict, device) -> dict:
        """{coord: tensor} of every active rank (padded all_gather)."""
        (coord, vec), = local.items()
        width = max(lengths.values()) if lengths else 0
        buf = torch.zeros(width, dtype=torch.float64, device=self.device)
        buf[: vec.numel()] = vec
        outs = [torch.empty_like(buf) for _ in range(self.rows * self.cols)]
        self._wait(self.dist.all_gather(outs, buf, group=self.active_group, async_op=True), "gather_vectors")
        return {(r // self.cols, r % self.cols): outs[r][: lengths[(r // self.cols, r % self.cols)]]
                for r in range(self.rows * self.cols)}

    def barrier(self):
        self.dist.barrier()


class PeerAxis:
    """One rank's side of a peer exchange on one axis: its receive buffer
    (2 parities x G slots x len doubles), arrival counter, epoch and CTA
    scratch, plus the IPC mappings of every group member's buffer and
    counter, packed as the C struct gridlp_peer_t."""

    def __init__(self, dist, group, members: list, my_slot: int, length: int, device, timeout: float = 120.0):
        from torch.multiprocessing.reductions import reduce_tensor

        from . import native

        G = len(members)
        self.recv = torch.zeros(max(2 * G * length, 1), dtype=torch.float64, device=device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        self.cta_count = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        mine = (reduce_tensor(self.recv), reduce_tensor(self.flag))
        got = [None] * G
        dist.all_gather_object(got, mine, group=group)
        self._mapped = []                      # keep the imported tensors (and their IPC mappings) alive
        c = native.Peer()
        for q, ((fr, fa), (gr, ga)) in enumerate(got):
            if q == my_slot:
                rt, ft = self.recv, self.flag
            else:
                rt, ft = fr(*fa), gr(*ga)
                self._mapped += [rt, ft]
                if rt.device != self.recv.device:       # another GPU: NVLink P2P from this device
                    native.load().call("gridlp_enable_peer_access", rt.device.index)
            c.dst[q] = rt.data_ptr()
            c.flag[q] = ft.data_ptr()
        c.recv, c.my_flag = self.recv.data_ptr(), self.flag.data_ptr()
        c.epoch, c.cta_count = self.epoch.data_ptr(), self.cta_count.data_ptr()
        c.group_size, c.my_slot, c.len = G, my_slot, length
        c.timeout_ns = int(timeout * 1e9)
        self.struct = c
        self.length = length


class PeerGrid(NcclGrid):
    """NcclGrid's process layout with in-kernel peer-memory exchanges for
    the vector sums (torch.distributed only moves the IPC handles at setup
    and the once-per-pass scalar table)."""

    kind = "peer"

    def __init__(self, rows: int, cols: int, device, timeout: float = 120.0):
        super().__init__(rows, cols, device, timeout)
        self.axes = {}

    def setup_axes(self, row_len: int, col_len: int):
        """Create the C-axis (grid row, vectors of m_i) and R-axis (grid
        column, vectors of n_j) exchanges of this rank; every rank calls it
        in the same order."""
        if not self.active:
            return
        i, j = self.coord
        for ii in range(self.rows):
            members = [ii * self.cols + jj for jj in range(self.cols)]
            if ii == i:
                self.axes["C"] = PeerAxis(self.dist, self.row_groups[ii], members, j, row_len, self.device,
                                          self.timeout)
        for jj in range(self.cols):
            members = [ii * self.cols + jj for ii in range(self.rows)]
            if jj == j:
                self.axes["R"] = PeerAxis(self.dist, self.col_groups[jj], members, i, col_len, self.device,
                                          self.timeout)

    def reduce(self, axis, index, partials, scratch=None):
        raise RuntimeError("PeerGrid sums inside the kernels; reduce() is never called")
