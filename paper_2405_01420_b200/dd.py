"""Spatial domain decomposition of the NB path over 2/4/8 GPUs.

Reference shape (/root/reference/pkg/src/mdgpusim/pipeline.py:267-438): near-cubic rank grid
`balanced_dims` (pipeline.py:42-60; 2 -> (2,1,1), 4 -> (2,2,1), 8 -> (2,2,2)), one halo pulse
per split dimension (pipeline.py:273-278, 363-380), the local force kernel overlapping the
coordinate halo (pipeline.py:344-349), the nonlocal kernel after the unpack
(pipeline.py:382-388) and the reverse force halo (pipeline.py:403-418).  There it is all
simulated time; here it is real:

  * one process per GPU, `torch.distributed` over NCCL; halo messages are stream-ordered
    point-to-point sends/receives batched per pulse (no host sync, unlike the paper's
    CPU-initiated MPI);
  * halo width = rlist_outer, staged pulses x -> y -> z forward edge/corner atoms;
  * half-shell import: a rank imports an atom of the domain at offset o (components in
    {-1, 0, 1} per split dimension, in domain units) iff the first non-zero component of o
    is +1.  For every cross-domain pair exactly one of o and -o qualifies, so each pair is
    computed exactly once, on one rank, as a plain home x halo pair of the nonlocal list (no
    masks, no halo-halo pairs).  In pulse d this means: send to the down neighbour the home
    and imported atoms near the lower face, and to the up neighbour only the imported atoms
    near the upper face (home atoms sent up would arrive with offset -1 in dimension d);
  * forces on imported atoms go back through the reverse pulses and are accumulated by
    the owner (z -> y -> x);
  * atoms are (re)assigned to domains at search steps from the global coordinates.

The per-rank engine is libnbx (`NbxEngine`); the host logic takes any object with the same
methods so the multi-process logic is also testable on CPU with gloo (tests/test_dd.py).
"""
from __future__ import annotations

import json
import math
import os
import time

import numpy as np


def balanced_dims(n: int):
    """Same factorisation as the reference's pipeline.balanced_dims (pipeline.py:42-60)."""
    if n < 1:
        raise ValueError("need at least one rank")
    best = (n, 1, 1)
    for dz in range(1, int(round(n ** (1 / 3))) + 1):
        if n % dz:
            continue
        rest = n // dz
        for dy in range(dz, int(rest**0.5) + 1):
            if rest % dy:
                continue
            dx = rest // dy
            if dx >= dy and (dx - dz) < (max(best) - min(best)):
                best = (dx, dy, dz)
    return best


def rank_coords(rank, dims):
    return (rank % dims[0], (rank // dims[0]) % dims[1], rank // (dims[0] * dims[1]))


def coords_rank(c, dims):
    return (c[0] % dims[0]) + dims[0] * ((c[1] % dims[1]) + dims[1] * (c[2] % dims[2]))


class NbxEngine:
    """Per-rank libnbx context with a local (home) and a nonlocal (halo) grid."""

    def __init__(self, system, device, pbc):
        import torch

        from . import nbx
        self.torch = torch
        self.nbx = nbx
        self.device = device
        self.params = nbx.make_params(**system.params())
        self.ctx = nbx.Context(self.params, device)
        q = np.ascontiguousarray(system.q, np.float32)
        t = np.ascontiguousarray(system.type, np.int32)
        c6c12 = np.ascontiguousarray(system.c6c12, np.float32)
        eo = np.ascontiguousarray(system.excl_offsets, np.int32)
        eg = np.ascontiguousarray(system.excl_gids, np.int32)
        L = nbx.lib()
        nbx.check(L.nbx_set_topology(self.ctx.h, system.natoms, nbx._ptr(q), nbx._ptr(t), int(c6c12.shape[0]),
                                     nbx._ptr(c6c12), nbx._ptr(eo), nbx._ptr(eg)))
        self.box = np.ascontiguousarray(system.box, np.float32)
        self.pbc = np.ascontiguousarray(pbc, np.int32)
        nbx.check(L.nbx_set_box(self.ctx.h, nbx._ptr(self.box), nbx._ptr(self.pbc)))

    def _st(self, stream=None):
        return self.nbx._stream(self.torch, stream)

    def grid_build(self, g, x, gid, lo, size):
        nbx = self.nbx
        lo = np.ascontiguousarray(lo, np.float32)
        size = np.ascontiguousarray(size, np.float32)
        n = int(x.shape[0])
        nbx.check(nbx.lib().nbx_grid_build(self.ctx.h, g, n, nbx._dev_ptr(x) if n else None,
                                           nbx._dev_ptr(gid) if n else None, nbx._ptr(lo), nbx._ptr(size),
                                           self._st()))

    def search(self, lst):
        self.nbx.check(self.nbx.lib().nbx_search(self.ctx.h, lst, self._st()))

    def grid_search_pair(self, x_home, gid_home, lo_l, size_l, x_halo, gid_halo, lo_n, size_n, side_stream):
        """Both grids and both lists of a DD search step, the halo half on side_stream."""
        nbx = self.nbx
        a = [np.ascontiguousarray(v, np.float32) for v in (lo_l, size_l, lo_n, size_n)]
        nh, nn = int(x_home.shape[0]), int(x_halo.shape[0])
        nbx.check(nbx.lib().nbx_grid_search_pair(
            self.ctx.h, nh, nbx._dev_ptr(x_home) if nh else None, nbx._dev_ptr(gid_home) if nh else None,
            nbx._ptr(a[0]), nbx._ptr(a[1]), nn, nbx._dev_ptr(x_halo) if nn else None,
            nbx._dev_ptr(gid_halo) if nn else None, nbx._ptr(a[2]), nbx._ptr(a[3]), self._st(),
            self._st(side_stream)))

    def put_x(self, g, x, stream=None):
        if x.shape[0]:
            self.nbx.check(self.nbx.lib().nbx_put_x(self.ctx.h, g, self.nbx._dev_ptr(x), self._st(stream)))

    def prune(self, lst, stream=None):
        self.nbx.check(self.nbx.lib().nbx_prune(self.ctx.h, lst, 0, 1, self._st(stream)))

    def force(self, lst, flags, stream=None):
        self.nbx.check(self.nbx.lib().nbx_force(self.ctx.h, lst, flags, self._st(stream)))

    def get_f(self, g, f, accumulate=False, stream=None):
        if f.shape[0]:
            self.nbx.check(self.nbx.lib().nbx_get_f(self.ctx.h, g, self.nbx._dev_ptr(f), 1 if accumulate else 0,
                                                    self._st(stream)))

    def clear_energies(self, stream=None):
        self.nbx.check(self.nbx.lib().nbx_clear_energies(self.ctx.h, self._st(stream)))

    def energies(self, stream=None):
        e = np.zeros(2)
        v = np.zeros(9)
        self.nbx.check(self.nbx.lib().nbx_energies(self.ctx.h, self.nbx._ptr(e), self.nbx._ptr(v), self._st(stream)))
        return e, v

    def count_pairs(self, lst):
        import ctypes as C
        p, s = C.c_int64(), C.c_int64()
        self.nbx.check(self.nbx.lib().nbx_count_pairs(self.ctx.h, lst, C.byref(p), C.byref(s), self._st()))
        return p.value, s.value

    def halo_pack(self, x, idx, shift, out, stream=None):
        nbx = self.nbx
        n = int(idx.shape[0])
        if n:
            sh = np.ascontiguousarray(shift, np.float32)
            nbx.check(nbx.lib().nbx_halo_pack_x(nbx._dev_ptr(x), nbx._dev_ptr(idx), n, nbx._ptr(sh),
                                                nbx._dev_ptr(out), self._st(stream)))

    def halo_unpack_add(self, f, idx, buf, stream=None):
        nbx = self.nbx
        n = int(idx.shape[0])
        if n:
            nbx.check(nbx.lib().nbx_halo_unpack_add_f(nbx._dev_ptr(f), nbx._dev_ptr(idx), n, nbx._dev_ptr(buf),
                                                      self._st(stream)))

    def launch_count(self):
        return self.nbx.lib().nbx_launch_count(self.ctx.h)

    # -- NVLink peer-memory halo (csrc/peer.cu) ------------------------------------------
    def peer_init(self, rank, world, capacity):
        h = np.zeros(64, np.uint8)
        self.nbx.check(self.nbx.lib().nbx_peer_init(self.ctx.h, rank, world, capacity, self.nbx._ptr(h)))
        return h

    def peer_open(self, handles):
        h = np.ascontiguousarray(handles, np.uint8)
        self.nbx.check(self.nbx.lib().nbx_peer_open(self.ctx.h, self.nbx._ptr(h)))

    def peer_set_halo(self, owner, home, shift):
        nbx = self.nbx
        n = int(owner.shape[0])
        nbx.check(nbx.lib().nbx_peer_set_halo(self.ctx.h, n, nbx._dev_ptr(owner) if n else None,
                                              nbx._dev_ptr(home) if n else None,
                                              nbx._dev_ptr(shift) if n else None, self._st()))

    def peer_put_x(self, x, seq, stream=None):
        self.nbx.check(self.nbx.lib().nbx_peer_put_x(self.ctx.h, self.nbx._dev_ptr(x) if x.shape[0] else None,
                                                     seq, self._st(stream)))

    def peer_halo_x(self, seq, stream=None):
        self.nbx.check(self.nbx.lib().nbx_peer_halo_x(self.ctx.h, seq, self._st(stream)))

    def peer_force_nonlocal(self, seq, flags=0, stream=None):
        self.nbx.check(self.nbx.lib().nbx_peer_force_nonlocal(self.ctx.h, seq, flags, self._st(stream)))

    def peer_get_f(self, f, seq, flags=0, stream=None):
        self.nbx.check(self.nbx.lib().nbx_peer_get_f(self.ctx.h, self.nbx._dev_ptr(f) if f.shape[0] else None,
                                                     seq, flags, self._st(stream)))

    def peer_repartition(self, geom, x_home, gid_home, rseq, x_ext, gid_ext, owner, home, shift):
        """nbx_peer_repartition: returns (overflowed, n_home, n_halo)."""
        import ctypes as C
        nbx = self.nbx
        nh, nhalo = C.c_int32(), C.c_int32()
        n = int(x_home.shape[0])
        code = nbx.lib().nbx_peer_repartition(
            self.ctx.h, C.byref(geom), nbx._dev_ptr(x_home) if n else None, nbx._dev_ptr(gid_home) if n else None,
            n, rseq, int(x_ext.shape[0]), nbx._dev_ptr(x_ext), nbx._dev_ptr(gid_ext), nbx._dev_ptr(owner),
            nbx._dev_ptr(home), nbx._dev_ptr(shift), C.byref(nh), C.byref(nhalo), self._st())
        if code not in (0, 4):  # 4 = NBX_ELIST_OVERFLOW: counts returned, caller falls back
            nbx.check(code)
        return code == 4, nh.value, nhalo.value

    def peer_status(self):
        import ctypes as C
        v = C.c_int32()
        self.nbx.check(self.nbx.lib().nbx_peer_status(self.ctx.h, C.byref(v)))
        return v.value

    def fma_peak(self):
        import ctypes as C
        v = C.c_double()
        self.nbx.check(self.nbx.lib().nbx_fma_peak(self.ctx.h, C.byref(v), self._st()))
        return v.value


class Pulse:
    __slots__ = ("dim", "down_peer", "up_peer", "down_idx", "up_idx", "shift_down", "shift_up",
                 "n_from_up", "n_from_down", "off_from_up", "off_from_down")


class DomainDecomposition:
    """One rank of the DD NB path.  `engine` is NbxEngine (GPU) or a test double."""

    def __init__(self, system, rank, world, engine_factory, device=None, group=None, halo="nccl"):
        import torch
        import torch.distributed as dist

        self.torch = torch
        self.dist = dist
        self.sys = system
        self.rank, self.world = rank, world
        self.group = group
        self.dims = balanced_dims(world)
        self.coord = rank_coords(rank, self.dims)
        self.box = np.asarray(system.box, np.float64)
        self.D = self.box / np.array(self.dims)
        self.rl = float(system.rlist_outer)
        for d in range(3):
            if self.dims[d] > 1 and self.D[d] < 2 * self.rl:
                raise ValueError(f"domain width {self.D[d]:.3f} nm < 2*rlist_outer in dim {d}")
        self.pbc = [1 if self.dims[d] == 1 else 0 for d in range(3)]
        self.device = device if device is not None else torch.device("cpu")
        self.engine = engine_factory(system, self.pbc)
        self.pulses = []
        self.n_home = 0
        self.n_ext = 0
        self.nstlist = system.nstlist
        self.prune_every = system.prune_every
        self.comm_stream = None
        if halo not in ("nccl", "p2p"):
            raise ValueError("halo must be 'nccl' or 'p2p'")
        self.halo = halo  # force-only steps: NCCL pulses, or NVLink peer memory (csrc/peer.cu)
        self.seq = 0
        self._peer_ready = False
        self.timing = None  # dict: host-side section times of repartition (tools/dd_repart_timing.py)
        self._t_last = 0.0
        self.profile_phases = False  # record per-phase CUDA events in step() (bench breakdown)
        self.phase_log = []
        # p2p steps: halo gather + nonlocal force on a side stream (NBX_DD_OVERLAP=0 disables)
        self.overlap_nonlocal = os.environ.get("NBX_DD_OVERLAP", "1") != "0"
        self._side = None
        self._ev_x = self._ev_nl = None
        self._peer_cap = 0
        self.rseq = 0             # device repartitions so far (peer-path search steps)
        self._rp = None           # device-repartition output buffers (capacity-sized)
        self._geom = None
        self.repartitions = {"global": 0, "device": 0, "fallback": 0}
        # gloo moves host tensors only: with CUDA tensors (e.g. several ranks sharing one GPU,
        # tests/test_dd_gpu.py's oversubscribed mode) every exchange is staged through host
        # memory; with NCCL the device tensors go straight onto the wire
        self._staged = dist.get_backend(group) == "gloo" and self.device.type == "cuda"

    # ---------------------------------------------------------------------- partitioning
    def _exchange(self, sends, recvs):
        """One batched NCCL/gloo point-to-point group: sends/recvs are (tensor, peer) lists.
        Staged (gloo + CUDA tensors): completes before returning, through host copies."""
        dist = self.dist
        sends = [(t, p) for t, p in sends if t.numel()]
        recvs = [(t, p) for t, p in recvs if t.numel()]
        if not sends and not recvs:
            return []
        if self._staged:
            hs = [(t.cpu(), p) for t, p in sends]
            hr = [(self.torch.empty(t.shape, dtype=t.dtype), p) for t, p in recvs]
            ops = [dist.P2POp(dist.isend, t, p, group=self.group) for t, p in hs]
            ops += [dist.P2POp(dist.irecv, t, p, group=self.group) for t, p in hr]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for (t, _), (h, _) in zip(recvs, hr):
                t.copy_(h)
            return []
        ops = [dist.P2POp(dist.isend, t, p, group=self.group) for t, p in sends]
        ops += [dist.P2POp(dist.irecv, t, p, group=self.group) for t, p in recvs]
        return dist.batch_isend_irecv(ops)

    def _all_reduce(self, t, op=None):
        """In-place all-reduce (host-staged under gloo with CUDA tensors)."""
        dist = self.dist
        op = dist.ReduceOp.SUM if op is None else op
        if self._staged:
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)
        return t

    def _all_gather(self, t):
        dist = self.dist
        src = t.cpu() if self._staged else t
        out = [self.torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(out, src, group=self.group)
        return out

    def _tick(self, name=None):
        if self.timing is None:
            return
        self.torch.cuda.synchronize()
        t = time.perf_counter()
        if name is not None:
            self.timing[name] = self.timing.get(name, 0.0) + (t - self._t_last)
        self._t_last = t

    def repartition(self, x_global=None, x_home=None):
        """A search step: (re)assign home atoms, build the halo plan, grids and lists.

        x_global given (every rank the same [N, 3] coordinates): the host-orchestrated global
        partition (first call, NCCL halo, fallback).  Otherwise, on the peer-memory path, the
        device-side neighbour-only repartition (nbx_peer_repartition) from this rank's current
        home coordinates x_home (default: those of the last step): no global coordinates, no
        per-pulse host synchronisation, two counts read at the end."""
        if x_global is None:
            if not (self.halo == "p2p" and self._peer_ready):
                raise ValueError("x_global is required for the first partition and for the NCCL halo path")
            return self._repartition_device(x_home)
        self.repartitions["global"] += 1
        return self._repartition_global(x_global)

    def _repartition_global(self, x_global):
        torch = self.torch
        dev = self.device
        self.check_peer()
        self._tick()
        box = torch.tensor(self.box, dtype=torch.float32, device=dev)
        xg = x_global.to(dev, torch.float32)
        xw = xg - torch.floor(xg / box) * box
        D = torch.tensor(self.D, dtype=torch.float32, device=dev)
        cidx = torch.clamp(torch.floor(xw / D).to(torch.int64), min=0)
        dims_t = torch.tensor(self.dims, dtype=torch.int64, device=dev)
        cidx = torch.minimum(cidx, dims_t - 1)
        owner = cidx[:, 0] + self.dims[0] * (cidx[:, 1] + self.dims[1] * cidx[:, 2])
        home = torch.nonzero(owner == self.rank).flatten()
        self.home_gid = home.to(torch.int32)
        if self.halo == "p2p":
            self._xw = xw
        self._tick("owners")
        self.n_home = int(home.numel())
        X = xw[home].contiguous()
        # per atom (global id, owner rank, index in the owner's home order), carried through
        # the pulses with the coordinates (the peer-memory halo addresses owners by it)
        M = torch.stack([self.home_gid, torch.full_like(self.home_gid, self.rank),
                         torch.arange(self.n_home, dtype=torch.int32, device=dev)], dim=1)
        lo = np.array([self.coord[d] * self.D[d] for d in range(3)])
        self.lo = lo
        self.pulses = []
        for d in range(3):
            n_d = self.dims[d]
            if n_d == 1:
                continue
            p = Pulse()
            p.dim = d
            c = list(self.coord)
            c[d] = self.coord[d] - 1
            p.down_peer = coords_rank(c, self.dims)
            c[d] = self.coord[d] + 1
            p.up_peer = coords_rank(c, self.dims)
            lo_d, hi_d = lo[d], lo[d] + self.D[d]
            # half-shell import: down-going messages carry home and imported atoms near the
            # lower face; up-going ones only imported atoms near the upper face (see header).
            # Both index sets come from one nonzero (one host sync); coordinates and the
            # (gid, owner, home index) metadata travel as one packed float32 [n, 6] message
            # per direction (the int32 metadata bit-cast), so a pulse is one count round trip
            # and one data round trip.
            down_m = X[:, d] < lo_d + self.rl
            up_m = X[:, d] >= hi_d - self.rl
            up_m[:self.n_home] = False
            # counts on the device, exchanged while the index sets are extracted; one host read
            # of all four counts after the single nonzero
            cnt_send = torch.stack([down_m.sum(), up_m.sum()]).to(torch.int64)
            cnt_from_up = torch.zeros(2, dtype=torch.int64, device=dev)
            cnt_from_down = torch.zeros(2, dtype=torch.int64, device=dev)
            works = self._exchange([(cnt_send, p.down_peer), (cnt_send, p.up_peer)],
                                   [(cnt_from_up, p.up_peer), (cnt_from_down, p.down_peer)])
            nz = torch.nonzero(torch.stack([down_m, up_m]))[:, 1].to(torch.int32)
            for w in works:
                w.wait()
            n_down, _, p.n_from_up, p.n_from_down = (
                int(v) for v in torch.stack([cnt_send[0], cnt_send[1], cnt_from_up[0], cnt_from_down[1]]).tolist())
            p.down_idx = nz[:n_down]
            p.up_idx = nz[n_down:]
            sd = np.zeros(3, np.float32)
            su = np.zeros(3, np.float32)
            if self.coord[d] == 0:
                sd[d] = self.box[d]
            if self.coord[d] == n_d - 1:
                su[d] = -self.box[d]
            p.shift_down, p.shift_up = sd, su
            n0 = X.shape[0]
            p.off_from_up, p.off_from_down = n0, n0 + p.n_from_up
            XM = torch.cat([X, M.view(torch.float32)], dim=1)  # [n, 6]: x, y, z | gid, owner, home
            send_d = XM[p.down_idx.long()]
            send_d[:, :3] += torch.from_numpy(sd).to(dev)
            send_u = XM[p.up_idx.long()]
            send_u[:, :3] += torch.from_numpy(su).to(dev)
            recv_u = torch.empty((p.n_from_up, 6), dtype=torch.float32, device=dev)
            recv_d = torch.empty((p.n_from_down, 6), dtype=torch.float32, device=dev)
            for w in self._exchange([(send_d, p.down_peer), (send_u, p.up_peer)],
                                    [(recv_u, p.up_peer), (recv_d, p.down_peer)]):
                w.wait()
            R = torch.cat([recv_u, recv_d])
            X = torch.cat([X, R[:, :3]])
            M = torch.cat([M, R[:, 3:].contiguous().view(torch.int32)])
            self.pulses.append(p)
            self._tick(f"pulse{d}")
        self.n_ext = X.shape[0]
        self.x_ext = X.contiguous()
        self.gid_ext = M[:, 0].contiguous()
        self._meta_halo = M[self.n_home:]
        self.f_ext = torch.zeros_like(self.x_ext)
        self.fbuf_down = [torch.empty((p.down_idx.numel(), 3), dtype=torch.float32, device=dev) for p in self.pulses]
        self.fbuf_up = [torch.empty((p.up_idx.numel(), 3), dtype=torch.float32, device=dev) for p in self.pulses]
        self.xbuf_down = [torch.empty((p.down_idx.numel(), 3), dtype=torch.float32, device=dev) for p in self.pulses]
        self.xbuf_up = [torch.empty((p.up_idx.numel(), 3), dtype=torch.float32, device=dev) for p in self.pulses]
        # grids: local = home atoms over the home domain (periodic only in undivided dims),
        # nonlocal = imported atoms over the domain grown by rlist in split dims
        size_l = np.array([self.D[d] if self.dims[d] > 1 else self.box[d] for d in range(3)], np.float32)
        lo_l = np.array([lo[d] if self.dims[d] > 1 else 0.0 for d in range(3)], np.float32)
        size_n = np.array([self.D[d] + 2 * self.rl if self.dims[d] > 1 else self.box[d] for d in range(3)], np.float32)
        lo_n = np.array([lo[d] - self.rl if self.dims[d] > 1 else 0.0 for d in range(3)], np.float32)
        self._tick("buffers")
        self._grids_and_searches(size_l, lo_l, size_n, lo_n)
        if self.halo == "p2p":
            self._peer_map()
            self._tick("peer_map")
        return self.n_home

    def _grids_and_searches(self, size_l, lo_l, size_n, lo_n):
        """Home grid + local list and halo grid + nonlocal list of a search step.  On the GPU
        engine both halves run overlapped, the halo half on the side stream
        (nbx_grid_search_pair; NBX_DD_PAIR_SEARCH=0 restores the four sequential calls)."""
        eng = self.engine
        xh, gh = self.x_ext[:self.n_home], self.gid_ext[:self.n_home]
        xn, gn = self.x_ext[self.n_home:], self.gid_ext[self.n_home:]
        if hasattr(eng, "grid_search_pair") and os.environ.get("NBX_DD_PAIR_SEARCH", "1") != "0":
            if self._side is None:
                self._side = self.torch.cuda.Stream(device=self.device)
            eng.grid_search_pair(xh, gh, lo_l, size_l, xn, gn, lo_n, size_n, self._side)
            self._tick("grids_searches")
        else:
            eng.grid_build(0, xh, gh, lo_l, size_l)
            self._tick("grid0")
            eng.search(0)
            self._tick("search0")
            eng.grid_build(1, xn, gn, lo_n, size_n)
            self._tick("grid1")
            eng.search(1)
            self._tick("search1")

    def dd_geom(self):
        """nbx_dd_geom of this rank: domain, neighbour ranks, half-shell import offsets."""
        if self._geom is not None:
            return self._geom
        import itertools

        from . import nbx
        g = nbx.DDGeom()
        box32 = np.asarray(self.box, np.float32)
        D32 = np.asarray(self.D, np.float32)  # the host path's float32 domain edge
        for d in range(3):
            g.box[d] = float(box32[d])
            g.dlen[d] = float(D32[d])
            g.lo[d] = float(np.float32(self.coord[d] * self.D[d]))
            g.hi[d] = float(np.float32((self.coord[d] + 1) * self.D[d]))
            g.dims[d] = self.dims[d]
            g.coord[d] = self.coord[d]
        g.rl = self.rl
        rng = [(-1, 0, 1) if self.dims[d] > 1 else (0,) for d in range(3)]
        srcs = []
        offs = []
        for o in itertools.product(*rng):
            c = [self.coord[d] + o[d] for d in range(3)]
            r = coords_rank(c, self.dims)
            if r not in srcs:
                srcs.append(r)
            nz = [v for v in o if v != 0]
            if nz and nz[0] == 1:
                sh = [box32[d] if c[d] >= self.dims[d] else (-box32[d] if c[d] < 0 else 0.0) for d in range(3)]
                offs.append((r, o, sh))
        g.n_src = len(srcs)
        for k, r in enumerate(srcs):
            g.src_rank[k] = r
        g.n_off = len(offs)
        for k, (r, o, sh) in enumerate(offs):
            g.off_rank[k] = r
            for d in range(3):
                g.off_dir[k][d] = o[d]
                g.off_shift[k][d] = float(sh[d])
        self._geom = g
        return g

    def _repartition_device(self, x_home=None):
        torch, dist = self.torch, self.dist
        dev = self.device
        self.check_peer()
        self._tick()
        x_home = (self.x_ext[:self.n_home] if x_home is None else x_home).contiguous()
        gid_home = self.home_gid.contiguous()
        B = self._rp
        if B is not None:
            # the inputs may be views of the output buffers (the previous repartition's
            # result): the library publishes them before writing the outputs, but an overflow
            # falls back to the global path, which needs the inputs intact -- copy them
            if x_home.data_ptr() >= B["x"].data_ptr() and x_home.data_ptr() < B["x"].data_ptr() + B["x"].nbytes:
                x_home = x_home.clone()
            if gid_home.data_ptr() >= B["gid"].data_ptr() and gid_home.data_ptr() < B["gid"].data_ptr() + B["gid"].nbytes:
                gid_home = gid_home.clone()
        cap_ext = 3 * self._peer_cap
        if self._rp is None or self._rp["x"].shape[0] < cap_ext:
            self._rp = {"x": torch.empty((cap_ext, 3), dtype=torch.float32, device=dev),
                        "gid": torch.empty(cap_ext, dtype=torch.int32, device=dev),
                        "owner": torch.empty(cap_ext, dtype=torch.int32, device=dev),
                        "home": torch.empty(cap_ext, dtype=torch.int32, device=dev),
                        "shift": torch.empty((cap_ext, 3), dtype=torch.float32, device=dev),
                        "f": torch.zeros((cap_ext, 3), dtype=torch.float32, device=dev)}
        B = self._rp
        self.rseq += 1
        over, nh, nhalo = self.engine.peer_repartition(self.dd_geom(), x_home, gid_home, self.rseq & 0xFFFFFFFF,
                                                       B["x"], B["gid"], B["owner"], B["home"], B["shift"])
        self._tick("device_repartition")
        chk = torch.tensor([nh, int(over)], dtype=torch.int64, device=dev)
        chk = self._all_reduce(chk).cpu()
        self._tick("conservation_check")
        if int(chk[1]) or int(chk[0]) != self.sys.natoms:
            # capacity overflow or lost atoms (moved more than one domain): rebuild globally from
            # an all-gather of the home sets (rare; the regions regrow in _peer_map)
            self.repartitions["fallback"] += 1
            return self._repartition_global(self._gather_global(x_home, gid_home))
        self.repartitions["device"] += 1
        self.n_home, self.n_ext = nh, nh + nhalo
        self.x_ext = B["x"][:self.n_ext]
        self.gid_ext = B["gid"][:self.n_ext]
        self.home_gid = self.gid_ext[:self.n_home]
        self.f_ext = B["f"][:self.n_ext]
        self.f_ext.zero_()
        self.pulses = []  # the message-passing halo plan is not built on this path
        size_l, lo_l, size_n, lo_n = self._grid_boxes()
        self._grids_and_searches(size_l, lo_l, size_n, lo_n)
        self._peer_owner = B["owner"][:nhalo]
        self._peer_home = B["home"][:nhalo]
        self._peer_shift = B["shift"][:nhalo]
        self.engine.peer_set_halo(self._peer_owner, self._peer_home, self._peer_shift)
        self._tick("peer_map")
        return self.n_home

    def _gather_global(self, x_home, gid_home):
        """All ranks' home sets -> the global [N, 3] coordinate array on every rank."""
        torch = self.torch
        dev = self.device
        n = torch.tensor([int(x_home.shape[0])], dtype=torch.int64, device=dev)
        ns = [int(v) for v in self._all_gather(n)]
        mx = max(ns)
        xp = torch.zeros((mx, 3), dtype=torch.float32, device=dev)
        gp = torch.zeros(mx, dtype=torch.int64, device=dev)
        xp[:ns[self.rank]] = x_home
        gp[:ns[self.rank]] = gid_home.long()
        xs, gs = self._all_gather(xp), self._all_gather(gp)
        xg = torch.empty((self.sys.natoms, 3), dtype=torch.float32, device=dev)
        seen = torch.zeros(self.sys.natoms, dtype=torch.int32, device=dev)
        for r in range(self.world):
            g = gs[r][:ns[r]].to(dev)
            xg[g] = xs[r][:ns[r]].to(dev)
            seen.index_add_(0, g, torch.ones_like(g, dtype=torch.int32))
        if not bool((seen == 1).all()):
            raise RuntimeError("DD fallback: the ranks' home sets do not partition the atoms")
        return xg

    def _grid_boxes(self):
        """(size, lo) of the local (home) grid and the nonlocal (halo) grid."""
        lo = np.array([self.coord[d] * self.D[d] for d in range(3)])
        size_l = np.array([self.D[d] if self.dims[d] > 1 else self.box[d] for d in range(3)], np.float32)
        lo_l = np.array([lo[d] if self.dims[d] > 1 else 0.0 for d in range(3)], np.float32)
        size_n = np.array([self.D[d] + 2 * self.rl if self.dims[d] > 1 else self.box[d] for d in range(3)], np.float32)
        lo_n = np.array([lo[d] - self.rl if self.dims[d] > 1 else 0.0 for d in range(3)], np.float32)
        return size_l, lo_l, size_n, lo_n

    def _peer_map(self):
        """Peer halo map after a repartition: for every imported atom its owner rank, its index
        in the owner's home order (home atoms are in increasing global id) and its import
        shift (a multiple of the box edge per dimension).

        The IPC regions hold `cap` home atoms per rank (the same on all ranks).  Every
        repartition all-reduces the largest home count; when a rank outgrows `cap` (load
        imbalance after atoms moved) all ranks re-create and re-exchange their regions at
        1.25x the new maximum, together, after their outstanding peer traffic has drained."""
        torch, dist = self.torch, self.dist
        dev = self.device
        nmax = torch.tensor([self.n_home], dtype=torch.int64, device=dev)
        nmax = int(self._all_reduce(nmax, op=dist.ReduceOp.MAX)[0])
        if not self._peer_ready or nmax > self._peer_cap:
            # capacity: 1.5x the mean home count (env NBX_PEER_CAP_FACTOR; tests shrink it to force
            # a regrow) and at least 1.25x the current largest home set
            fac = float(os.environ.get("NBX_PEER_CAP_FACTOR", "1.5"))
            cap = max(int(math.ceil(fac * self.sys.natoms / self.world)) + 4096, int(math.ceil(1.25 * nmax)))
            if self._peer_ready:
                torch.cuda.synchronize(dev)  # nobody still reads / reduces into the old regions
                dist.barrier(group=self.group)
            h = self.engine.peer_init(self.rank, self.world, cap)
            hs = self._all_gather(torch.from_numpy(h).to(dev))
            self.engine.peer_open(torch.cat([t.cpu() for t in hs]).numpy())
            self._peer_ready = True
            self._peer_cap = cap
            self.peer_inits = getattr(self, "peer_inits", 0) + 1
        m = self._meta_halo
        box = torch.tensor(self.box, dtype=torch.float32, device=dev)
        sh = torch.round((self.x_ext[self.n_home:] - self._xw[m[:, 0].long()]) / box) * box
        self._peer_owner = m[:, 1].contiguous()
        self._peer_home = m[:, 2].contiguous()
        self._peer_shift = sh.to(torch.float32).contiguous()
        self.engine.peer_set_halo(self._peer_owner, self._peer_home, self._peer_shift)
        self._xw = None
        # every rank's map and regions are in place before anyone's next signal
        dist.barrier(group=self.group)

    def check_peer(self):
        """Raise if a peer-memory wait timed out (a rank stopped taking steps) or the halo map
        pointed outside the peer regions."""
        if self.halo == "p2p" and self._peer_ready:
            st = self.engine.peer_status()
            if st == 1:
                raise RuntimeError("peer-memory halo: a wait for another rank timed out")
            if st:
                raise RuntimeError("peer-memory halo: invalid halo map (owner / home index out of range)")

    # ---------------------------------------------------------------------- per step
    def halo_x(self):
        """Coordinate halo: pack with shift, exchange per pulse, received straight in place."""
        eng = self.engine
        works = []
        for k, p in enumerate(self.pulses):
            for w in works:
                w.wait()  # pulse k forwards atoms received in pulse k-1
            eng.halo_pack(self.x_ext, p.down_idx, p.shift_down, self.xbuf_down[k])
            eng.halo_pack(self.x_ext, p.up_idx, p.shift_up, self.xbuf_up[k])
            ru = self.x_ext[p.off_from_up:p.off_from_up + p.n_from_up]
            rd = self.x_ext[p.off_from_down:p.off_from_down + p.n_from_down]
            works = self._exchange([(self.xbuf_down[k], p.down_peer), (self.xbuf_up[k], p.up_peer)],
                                   [(ru, p.up_peer), (rd, p.down_peer)])
        return works

    def halo_f(self):
        """Force halo: reverse pulses z -> y -> x, accumulated into the owner's atoms."""
        eng = self.engine
        for k in range(len(self.pulses) - 1, -1, -1):
            p = self.pulses[k]
            fu = self.f_ext[p.off_from_up:p.off_from_up + p.n_from_up]
            fd = self.f_ext[p.off_from_down:p.off_from_down + p.n_from_down]
            for w in self._exchange([(fu, p.up_peer), (fd, p.down_peer)],
                                    [(self.fbuf_down[k], p.down_peer), (self.fbuf_up[k], p.up_peer)]):
                w.wait()
            eng.halo_unpack_add(self.f_ext, p.down_idx, self.fbuf_down[k])
            eng.halo_unpack_add(self.f_ext, p.up_idx, self.fbuf_up[k])

    def step(self, x_home=None, step=1, energy=False, virial=False, prune=None):
        """One NB-path step: returns f_home (a view of the rank's force buffer, overwritten by
        the next step) and, with energy/virial, the all-reduced (energies, virial)."""
        eng = self.engine
        ev = self._events() if self.profile_phases else None
        if prune is None:
            prune = bool(self.prune_every) and step % self.prune_every == 0
        if self.halo == "p2p":
            return self._step_p2p(x_home, prune, ev, (1 if energy else 0) | (2 if virial else 0))
        if x_home is not None:
            self.x_ext[:self.n_home].copy_(x_home)
        if ev:
            ev[0].record()
        works = self.halo_x()  # NCCL in flight while the local kernel runs
        eng.put_x(0, self.x_ext[:self.n_home])
        if prune:
            eng.prune(0)
        flags = (1 if energy else 0) | (2 if virial else 0)
        if flags:
            eng.clear_energies()
        eng.force(0, flags)
        if ev:
            ev[1].record()
        for w in works:
            w.wait()
        if ev:
            ev[2].record()
        eng.put_x(1, self.x_ext[self.n_home:])
        if prune:
            eng.prune(1)
        eng.force(1, flags)
        if ev:
            ev[3].record()
        res = None
        if flags:
            res = self._reduce_energies()
        eng.get_f(0, self.f_ext[:self.n_home])
        eng.get_f(1, self.f_ext[self.n_home:])
        self.halo_f()
        if ev:
            ev[4].record()
            self.phase_log.append(ev)
        f_home = self.f_ext[:self.n_home]
        return (f_home, res) if res is not None else f_home

    def _reduce_energies(self):
        """This rank's (E, virial) share -> all-reduced totals (host arrays)."""
        e, v = self.engine.energies()
        t = self.torch.tensor(np.concatenate([e, v]), dtype=self.torch.float64, device=self.device)
        t = self._all_reduce(t).cpu().numpy()
        return t[:2], t[2:].reshape(3, 3)

    def _step_p2p(self, x_home, prune, ev, flags=0):
        """A step with the NVLink peer-memory halo: no messages, no pack/unpack, no reverse
        pulses (csrc/peer.cu).  flags (1 energy, 2 virial): the nonlocal kernel accumulates
        energies, and the virial's x (x) f is summed per grid before the forces move (halo
        atoms before the push to their owners, home atoms before the inbox is added), so
        energy / virial steps take the same halo as force-only ones.  x_home=None: the
        coordinates of the last repartition (or of the last step)."""
        eng = self.engine
        self.seq += 1
        seq = self.seq & 0xFFFFFFFF
        x = self.x_ext[:self.n_home] if x_home is None else x_home.contiguous()
        if flags:
            eng.clear_energies()
        if ev:
            ev[0].record()
        eng.peer_put_x(x, seq)  # grid-0 X op + publish + signal
        if self.overlap_nonlocal and not ev:
            # halo gather + nonlocal force on a side stream: they start as soon as the owners
            # have published and overlap the local kernel's tail (the two lists use separate
            # work counters; both red.add into the home cluster forces)
            torch = self.torch
            main = torch.cuda.current_stream()
            if self._side is None:
                self._side = torch.cuda.Stream(device=self.device)
            if self._ev_x is None:
                self._ev_x = torch.cuda.Event()
                self._ev_nl = torch.cuda.Event()
            self._ev_x.record(main)
            with torch.cuda.stream(self._side):
                self._side.wait_event(self._ev_x)
                eng.peer_halo_x(seq)
                if prune:
                    eng.prune(1)
                eng.peer_force_nonlocal(seq, flags)
                self._ev_nl.record(self._side)
            if prune:
                eng.prune(0)
            eng.force(0, flags)
            main.wait_event(self._ev_nl)
            f_home = self.f_ext[:self.n_home]
            eng.peer_get_f(f_home, seq, flags)  # wait for the senders, home forces + inbox
        else:
            if prune:
                eng.prune(0)
            eng.force(0, flags)
            if ev:
                ev[1].record()
            eng.peer_halo_x(seq)  # wait for the owners, gather the halo over NVLink
            if ev:
                ev[2].record()
            if prune:
                eng.prune(1)
            eng.peer_force_nonlocal(seq, flags)  # j forces straight into the owners' inboxes
            if ev:
                ev[3].record()
            f_home = self.f_ext[:self.n_home]
            eng.peer_get_f(f_home, seq, flags)  # wait for the senders, home forces + inbox
            if ev:
                ev[4].record()
                self.phase_log.append(ev)
        if flags:
            return f_home, self._reduce_energies()
        return f_home

    def _events(self):
        E = self.torch.cuda.Event
        return [E(enable_timing=True) for _ in range(5)]

    def phase_summary(self):
        """Mean ms per step of: local (halo issue + local force), halo wait (exposed x halo),
        nonlocal force, F ops + force halo; from the events of profiled steps."""
        self.torch.cuda.synchronize()
        if not self.phase_log:
            return None
        names = ["local", "x_halo_exposed", "nonlocal", "f_ops_and_f_halo"]
        acc = [0.0] * 4
        for ev in self.phase_log:
            for k in range(4):
                acc[k] += ev[k].elapsed_time(ev[k + 1])
        return {n: a / len(self.phase_log) for n, a in zip(names, acc)}

    def count_pairs(self):
        p0, s0 = self.engine.count_pairs(0)
        p1, s1 = self.engine.count_pairs(1)
        return p0 + p1, s0 + s1


# ---------------------------------------------------------------------------- bench, N > 1
def bench(args, METRIC, UNIT, FLOPS_PER_PAIR, DESC, ClockSampler, time_cpu_port, load_traffic,
          step_kind=None, compose_era=None, motion_velocities=None, motion_sign=None):
    """N > 1 arm of bench.py: same cadence, window and era composition as the 1-GPU arm
    (bench.compose_era: the window starts with a search step = repartition + search, each
    rank composes one nstlist era from its per-kind step means, the max over ranks is the
    step time) and the same motion (x += sign v dt between steps on the home atoms; search
    steps repartition the moved global coordinates)."""
    import torch
    import torch.distributed as dist

    from . import systems
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    s = systems.make(args.config)
    halo = os.environ.get("NBX_DD_HALO", "p2p")
    dd = DomainDecomposition(s, rank, world, lambda sy, pbc: NbxEngine(sy, local, pbc), device=dev, halo=halo)
    xg0 = torch.from_numpy(s.x).to(dev)
    dt_ps = s.dt_fs * 1e-3
    vel = torch.from_numpy(motion_velocities(s.natoms, s.nstlist, dt_ps)).to(dev)
    net = [0.0]  # net forward motion steps of the global coordinates (every rank the same)

    def xg_now():
        return xg0 + vel * (net[0] * dt_ps)

    def move_home(xh, step):
        sg = motion_sign(step, s.nstlist)
        net[0] += sg
        return xh + vel[dd.home_gid.long()] * (sg * dt_ps)

    peak = dd.engine.fma_peak()

    def search_step_repartition(x_home):
        # peer path: the device-side neighbour-only repartition from the home coordinates;
        # NCCL path: the global partition from the (moved) global coordinates
        if halo == "p2p":
            return dd.repartition(x_home=x_home)
        return dd.repartition(xg_now())

    dd.repartition(xg_now())  # setup: first search sizes the lists and the single-pass buffers
    dd.step(None, step=0, prune=False)
    search_step_repartition(dd.x_ext[:dd.n_home])
    dd.step(None, step=0, prune=False)
    search_step_repartition(dd.x_ext[:dd.n_home])
    x_home = dd.x_ext[:dd.n_home].clone()
    for k in range(args.warmup):
        step = max(1, s.nstlist - args.warmup + k)
        x_home = move_home(x_home, step)
        dd.step(x_home, step=step)
    torch.cuda.synchronize()

    K = args.steps
    st = torch.cuda.current_stream()
    kinds = [step_kind(k, s.nstlist, s.prune_every) for k in range(K)]
    # clocks sampled by rank 0 only, every 250 ms: each nvidia-smi poll takes NVML locks that a
    # rank's CUDA calls can wait on, and search steps synchronise with the host
    clocks = ClockSampler(local, interval_ms=250,
                          enabled=(rank == 0 and os.environ.get("NBX_BENCH_CLOCKS", "1") != "0")).start()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = dd.engine.launch_count()
    a0 = dd.engine.nbx.lib().nbx_alloc_count()
    seg0 = torch.cuda.memory_stats(dev).get("segment.all.allocated", 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    e0.record(st)
    rep_cpu_ms = []  # host time of each repartition call on this rank (diagnostics)
    pairs_tot = slots_tot = None
    for k in range(K):
        if k:
            x_home = move_home(x_home, k)
        evs[k][0].record(st)
        if kinds[k] == "search":
            tc = time.perf_counter()
            search_step_repartition(x_home)
            rep_cpu_ms.append(1e3 * (time.perf_counter() - tc))
            x_home = dd.x_ext[:dd.n_home].clone()
            dd.step(None, step=k, prune=False)
        else:
            dd.step(x_home, step=k)
        evs[k][1].record(st)
    e1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    dd.check_peer()
    launches = dd.engine.launch_count() - l0
    allocs = dd.engine.nbx.lib().nbx_alloc_count() - a0
    segs = torch.cuda.memory_stats(dev).get("segment.all.allocated", 0) - seg0
    al = torch.tensor([allocs, segs], dtype=torch.int64, device=dev)
    al_all = [torch.zeros_like(al) for _ in range(world)]
    dist.all_gather(al_all, al)
    allocs_per_rank = [[int(v) for v in a.tolist()] for a in al_all]
    step_ms = [a.elapsed_time(b) for a, b in evs]
    era_ms, kind_ms, kind_n = compose_era(step_ms, kinds, s.nstlist, s.prune_every)
    t = torch.tensor([era_ms, e0.elapsed_time(e1) / K], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, window_max = float(t[0]), float(t[1])
    pairs, slots = dd.count_pairs()
    pt = torch.tensor([pairs, slots], dtype=torch.float64, device=dev)
    dist.all_reduce(pt)
    pairs_tot, slots_tot = float(pt[0]), float(pt[1])
    clk = clocks.stop()
    rc = torch.tensor(rep_cpu_ms or [0.0], dtype=torch.float64, device=dev)
    rc_all = [torch.zeros_like(rc) for _ in range(world)]
    dist.all_gather(rc_all, rc)
    rep_cpu_all = [[round(float(v), 1) for v in r] for r in rc_all]
    # per-phase breakdown on 10 extra (untimed) steps, all ranks starting together
    dist.barrier()
    torch.cuda.synchronize()
    dd.profile_phases = True
    for k in range(10):
        dd.step(x_home, step=1)
    phases = dd.phase_summary()
    dd.profile_phases = False
    # e2e: every step copies this rank's home coordinates from pinned host memory and reads
    # its home forces back (the public DomainDecomposition.step API; no search steps)
    e2e = None
    if not args.no_e2e:
        xh = x_home.cpu().pin_memory()
        fh = torch.empty((dd.n_home, 3), dtype=torch.float32).pin_memory()
        xd = torch.empty_like(x_home)
        Ke = max(1, min(K, 50))
        dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        for k in range(Ke):
            xd.copy_(xh, non_blocking=True)
            fo = dd.step(xd, step=1 + k)
            fh.copy_(fo, non_blocking=True)
        a1.record(st)
        torch.cuda.synchronize()
        dd.check_peer()
        te = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nb = torch.tensor([xh.numel() * 4, fh.numel() * 4], dtype=torch.float64, device=dev)
        dist.all_reduce(nb)
        # non-search steps only: add this arm's amortised search cost (the timed window's
        # search-step mean minus its plain-step mean, / nstlist) so the era matches `value`
        extra = (kind_ms.get("search", 0.0) - kind_ms.get("plain", 0.0)) / s.nstlist
        e_ms = float(te[0]) / Ke + max(extra, 0.0)
        e2e = {"value": pairs_tot / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(nb[0]), "d2h_bytes_per_step": int(nb[1]), "steps": Ke,
               "ms_per_step": e_ms, "ms_per_step_nonsearch": float(te[0]) / Ke,
               "api": "paper_2405_01420_b200.dd.DomainDecomposition.step (ctypes -> libnbx.so C-ABI), "
                      "all ranks, max over ranks; + amortised search step of the timed window"}
    if rank == 0:
        ms_per_step = ms_max
        value = pairs_tot / (ms_per_step * 1e-3)
        fl = FLOPS_PER_PAIR[s.coulomb] + {"comb-geom": 2, "comb-lb": 8}.get(s.lj_modifier, 0)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {DESC[args.config]}", "natoms": s.natoms,
                       "parallelism": f"spatial DD {dd.dims[0]}x{dd.dims[1]}x{dd.dims[2]}, "
                       + ("NVLink peer-memory halo (fused into X op / nonlocal force / F op)" if halo == "p2p"
                          else "NCCL P2P halo"),
                       "nstlist": s.nstlist, "prune_every": s.prune_every,
                       "l2": "inputs larger than L2" if s.natoms > 2_000_000 else "per-rank inputs may fit L2",
                       "step_time": "one nstlist era composed from each rank's per-kind step means, max over "
                                    "ranks; the window starts with a search (repartition) step",
                       "motion": "x += v dt between steps (v reversed every nstlist steps)",
                       "repartition": ("device-side neighbour-only (nbx_peer_repartition) from home coordinates"
                                       if halo == "p2p" else "global (host-orchestrated, NCCL pulses)")},
            "steps_per_s": 1e3 / ms_per_step, "ns_per_day": 86.4 * s.dt_fs / ms_per_step,
            "pairs_per_step": pairs_tot, "pair_slots_per_step": slots_tot,
            "roofline": {"bound": "fp32", "achieved": value / 1e12 * fl / world, "peak": peak, "unit": "TFLOP/s",
                         "frac": value / 1e12 * fl / world / peak, "traffic": load_traffic(args.config, world),
                         "note": "per GPU, whole NB step (not kernel-only) at N>1"},
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
            "device_allocs_in_timed_region_per_rank": allocs_per_rank,  # [libnbx, torch segments]
            "step_ms_rank0": {"era": era_ms, "by_kind": kind_ms, "kind_counts": kind_n,
                              "window_mean_max_over_ranks": window_max},
            "dd_phases_ms_rank0": phases,
            "repartition_host_ms_per_rank": rep_cpu_all,
            "repartitions_rank0": dict(dd.repartitions),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
