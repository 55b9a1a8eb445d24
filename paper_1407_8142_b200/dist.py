"""Sharded wavelet-tree build over P GPUs.

One process per GPU holds a contiguous chunk S_r of S.  The build has one
real exchange step (an MSD radix exchange on the top tau = min(8, L) bits):

1. every rank counts the top-tau digit of its chunk (``wt_digit_counts``,
   which also validates S[i] < sigma); the counts are all-gathered;
2. levels 0..tau-1: each rank builds the top levels of its own chunk
   (``wt_digits`` + ``wt_build`` on the digits); in the global level k the
   class p run (S_k is S stably sorted by its top k bits) is
   the concatenation, in rank order, of every rank's class-p run, placed at
   C_k(p) + (earlier ranks' class-p counts) -- the split-then-merge of
   PAPER.md:266-273 with the merge replaced by placement;
3. levels tau..L-1: every rank stably partitions its chunk by digit
   (``wt_partition``), an all-to-all sends each digit range to its owner,
   the owner partitions the received runs again (digit, then source rank,
   then position = S_tau restricted to its range) and builds them with
   ``wt_build``; level l >= tau of that local tree is the global level l at
   offset R_o (the elements with smaller digits);
4. the runs of steps 2-3 and the owners' node tables are all-gathered and
   placed with ``wt_gather_bits`` into a tree made by ``wt_create``;
   ``wt_finish`` computes the rank directory.  Every rank ends with the
   complete tree (bit-identical to the single-GPU build of S).

Collectives go through ``TorchComm`` (torch.distributed: NCCL on GPUs, gloo on
CPU for the host-logic tests); the local steps through ``CudaOps`` (the C ABI,
every element-level step in the library's kernels).  Both are parameters so
that the orchestration can be tested with other implementations.
"""
from __future__ import annotations

import numpy as np
import torch

from . import wt as _wt

TAU = 8  # levels per exchange digit (the group pass width)


def _levels(sigma: int) -> int:
    return (int(sigma) - 1).bit_length()


def _wpl(n: int) -> int:
    return ((int(n) + 511) // 512) * 8


def _bytes(t: torch.Tensor) -> torch.Tensor:
    if t.numel() == 0:
        return torch.zeros(0, dtype=torch.uint8, device=t.device)
    return t.contiguous().view(-1).view(torch.uint8)


def _as(b: torch.Tensor, dtype) -> torch.Tensor:
    """Byte tensor -> dtype (empty-safe)."""
    if b.numel() == 0:
        return torch.zeros(0, dtype=dtype, device=b.device)
    return b.contiguous().view(dtype)


class TorchComm:
    """Collectives over a torch.distributed process group (tensors of any
    dtype are moved as bytes, so NCCL never sees an unsupported dtype)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group))

    def all_gather(self, t: torch.Tensor) -> list:
        b = _bytes(t)
        out = [torch.empty_like(b) for _ in range(self.world)]
        self.dist.all_gather(out, b, group=self.group)
        return [o.view(t.dtype).view(t.shape) for o in out]

    def all_gather_v(self, t: torch.Tensor) -> list:
        """1-D tensors of different lengths."""
        b = _bytes(t)
        ns = [int(x) for x in self.all_gather(torch.tensor([b.numel()], dtype=torch.int64, device=t.device))]
        m = max(max(ns), 1)
        buf = torch.zeros(m, dtype=torch.uint8, device=t.device)
        buf[:b.numel()] = b
        outs = self.all_gather(buf)
        return [_as(o[:k], t.dtype) for o, k in zip(outs, ns)]

    def all_to_all_v(self, t: torch.Tensor, send_counts: list) -> torch.Tensor:
        """Send t[sum(send_counts[:j]) : +send_counts[j]] to rank j; returns
        what every rank sent here, concatenated in rank order."""
        eb = t.element_size()
        sc = torch.tensor([int(c) for c in send_counts], dtype=torch.int64, device=t.device)
        allc = [x.tolist() for x in self.all_gather(sc)]
        recv = [int(allc[j][self.rank]) for j in range(self.world)]
        b = _bytes(t)
        out = torch.empty(sum(recv) * eb, dtype=torch.uint8, device=t.device)
        sb, rb = [int(c) * eb for c in send_counts], [c * eb for c in recv]
        # the same collective on every backend (NCCL on GPUs, gloo in the CPU tests)
        self.dist.all_to_all_single(out, b, rb, sb, group=self.group)
        return _as(out, t.dtype)


class CudaOps:
    """Local steps through the C ABI (libwt_b200.so)."""

    def digit_counts(self, S, sigma, shift, tau):
        return _wt.digit_counts(S, sigma, shift, tau)

    def digits(self, S, shift, tau):
        return _wt.digits(S, shift, tau)

    def partition(self, S, shift, tau):
        return _wt.partition(S, shift, tau)

    def build(self, S, sigma):
        return _wt.build(S, sigma)

    def create(self, n, sigma, elem_bytes, total_nodes, device):
        return _wt.create(n, sigma, elem_bytes, total_nodes, device)

    def gather_bits(self, src, segs, dst):
        _wt.gather_bits(src, segs, dst)

    def finish(self, tree):
        _wt.finish(tree)


def _i64(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int64) if t.dtype == torch.uint64 else t


def _i32(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int32) if t.dtype == torch.uint32 else t


def plan_owners(D: np.ndarray, P: int) -> np.ndarray:
    """Owner of every top digit: contiguous digit ranges balanced by count
    (owner(d) = floor(P * start(d) / n), non-decreasing in d)."""
    n = int(D.sum())
    start = np.concatenate(([0], np.cumsum(D)[:-1])).astype(np.int64)
    if n == 0:
        return np.zeros(D.size, dtype=np.int64)
    return np.minimum(P - 1, (start * P) // n)


class ShardedPart:
    """One rank's share of a sharded build (``build_sharded(..., gather=False)``),
    before any bitmap crosses the interconnect:

    * ``top``: the tree of this rank's chunk over the top ``tau`` digit bits;
      its level k < tau run of class p is the global level-k run of class p
      restricted to this rank, placed at ``C_k(p)`` + the earlier ranks' class-p
      counts (``place_top`` gives those offsets);
    * ``deep``: the owner's tree of the elements whose top digit it owns (a
      contiguous digit range), in S_tau order; its level l >= tau is the
      global level l on positions ``[R_o, R_o + n_o)``, its nodes the global
      nodes of those levels with starts shifted by ``R_o``;
    * ``C``: every rank's digit counts (rank x digit), ``owner``: the owner of
      every digit.

    Every global bitmap bit and node is held by exactly one rank; ``assemble``
    (the all-gather of step 4) turns the parts into the complete tree."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    def place_top(self, k: int) -> dict:
        """{class p: (global offset of this rank's run, length)} of level k < tau."""
        w = self.tau - k
        out = {}
        for p in range(1 << k):
            lo_d, hi_d = p << w, (p + 1) << w
            c = int(self.C[self.rank, lo_d:hi_d].sum())
            if c:
                out[p] = (int(self.dstart[lo_d]) + int(self.C[:self.rank, lo_d:hi_d].sum()), c)
        return out

    def free(self):
        for t in (self.top, self.deep):
            if t is not None and hasattr(t, "free"):
                t.free()
        self.top = self.deep = None


def build_sharded(S_local: torch.Tensor, sigma: int, comm=None, ops=None, gather: bool = True,
                  exchange: bool = False):
    """Build the wavelet tree of S = concat over ranks of S_local (rank order).

    Collective: every rank of ``comm`` must call it.  With ``gather`` (the
    default) every rank returns the complete tree (a ``WaveletTree`` with the
    CUDA ops); without, every rank returns its ``ShardedPart`` (distributed
    output: no bitmap is all-gathered; ``assemble`` does it on demand).
    ``exchange`` runs the exchange steps even on a single rank (a one-rank
    process group then carries the same all_to_all_single / all_gather calls
    as P > 1; the tests use it to execute the NCCL path on one GPU)."""
    part = _build_parts(S_local, sigma, comm, ops, exchange)
    if not isinstance(part, ShardedPart):
        return part
    return assemble(part, comm, ops) if gather else part


def _build_parts(S_local: torch.Tensor, sigma: int, comm=None, ops=None, exchange: bool = False):
    comm = comm if comm is not None else TorchComm()
    ops = ops if ops is not None else CudaOps()
    P, r = comm.world, comm.rank
    S_local = S_local.contiguous().view(-1)
    if P == 1 and not exchange:  # nothing to exchange: the single-GPU build
        return ops.build(S_local, sigma)
    dev = S_local.device
    eb = S_local.element_size()
    L = _levels(sigma)
    ns = [int(x) for x in comm.all_gather(torch.tensor([S_local.numel()], dtype=torch.int64, device=dev))]
    n = sum(ns)
    tau = min(TAU, L) if L else 1
    shift = L - tau if L else 0
    ndig = 1 << tau

    # ---- 1: digit counts + validation, agreed by all ranks ----
    err = 0
    try:
        cnt = _i64(ops.digit_counts(S_local, sigma, shift, tau))
    except _wt.WtError as e:
        cnt, err = torch.zeros(ndig, dtype=torch.int64, device=dev), e.code
    meta = torch.cat([cnt, torch.tensor([err], dtype=torch.int64, device=dev)])
    allm = torch.stack(comm.all_gather(meta)).cpu().numpy()
    bad = [int(e) for e in allm[:, ndig] if e]
    if bad:
        raise _wt.WtError(bad[0], "build_sharded")
    C = allm[:, :ndig].astype(np.int64)  # C[rank, digit]
    if L == 0:
        t = ops.create(n, sigma, eb, 0, dev)
        ops.finish(t)
        return t
    D = C.sum(0)
    dstart = np.concatenate(([0], np.cumsum(D)[:-1])).astype(np.int64)
    W = _wpl(n)
    owner = plan_owners(D, P)

    # ---- 2: top levels of every chunk ----
    Tl = ops.build(ops.digits(S_local, shift, tau), ndig)

    # ---- 3: exchange by digit, owners build levels >= tau ----
    no = np.zeros(P, dtype=np.int64)
    To, R_o, n_o = None, 0, 0
    if L > tau:
        for o in range(P):
            no[o] = int(D[owner == o].sum())
        Sp = ops.partition(S_local, shift, tau)
        send = [int(C[r, owner == o].sum()) for o in range(P)]
        Rv = comm.all_to_all_v(Sp, send)
        del Sp
        Ro = ops.partition(Rv, shift, tau)
        del Rv
        n_o = Ro.numel()
        assert n_o == no[r]
        R_o = int(dstart[np.argmax(owner == r)]) if n_o else 0
        if n_o:
            To = ops.build(Ro, sigma)
    return ShardedPart(rank=r, world=P, n=n, ns=ns, sigma=sigma, eb=eb, L=L, tau=tau, C=C, D=D, dstart=dstart,
                       owner=owner, no=no, top=Tl, deep=To, R_o=R_o, n_o=n_o, device=dev)


def assemble(part: ShardedPart, comm=None, ops=None):
    """Step 4 of the sharded build: all-gather every rank's runs and nodes and
    place them into the complete tree (on every rank)."""
    comm = comm if comm is not None else TorchComm()
    ops = ops if ops is not None else CudaOps()
    P, r, n, ns, sigma, eb = part.world, part.rank, part.n, part.ns, part.sigma, part.eb
    L, tau, C, D, dstart, owner, no, dev = (part.L, part.tau, part.C, part.D, part.dstart, part.owner,
                                           part.no, part.device)
    W = _wpl(n)
    top_parts = comm.all_gather_v(_i64(part.top.bits).contiguous())
    deep_parts, node_parts = [], []
    if L > tau:
        To, R_o, n_o = part.deep, part.R_o, part.n_o
        if n_o:
            wo = _wpl(n_o)
            deep = _i64(To.bits)[tau * wo:].contiguous()
            lnp = _i64(To.level_node_ptr).cpu().numpy()
            lo = int(lnp[tau])
            keys = _i32(To.node_key)[lo:].to(torch.int64)
            starts = _i32(To.node_start)[lo:].to(torch.int64) + R_o
            packed = torch.stack([keys, starts], 1).reshape(-1)
            lcnt = torch.from_numpy(np.diff(lnp[tau:]).astype(np.int64)).to(dev)
        else:
            deep = torch.zeros(0, dtype=torch.int64, device=dev)
            packed = torch.zeros(0, dtype=torch.int64, device=dev)
            lcnt = torch.zeros(L - tau, dtype=torch.int64, device=dev)
        deep_parts = comm.all_gather_v(deep)
        node_parts = [p.view(-1, 2) for p in comm.all_gather_v(packed)]
        node_cnts = [c.cpu().numpy() for c in comm.all_gather(lcnt)]  # [owner][level - tau]
    part.free()

    # ---- 4: place every run, assemble the node table ----
    parts = top_parts + deep_parts
    base = np.concatenate(([0], np.cumsum([p.numel() for p in parts]))).astype(np.int64)
    segs = []
    for k in range(tau):
        w = tau - k
        for p in range(1 << k):
            lo_d, hi_d = p << w, (p + 1) << w
            run = int(dstart[lo_d])
            for rr in range(P):
                c = int(C[rr, lo_d:hi_d].sum())
                if c:
                    lstart = int(C[rr, :lo_d].sum())
                    segs.append((k * W * 64 + run, int(base[rr]) * 64 + k * _wpl(ns[rr]) * 64 + lstart, c))
                    run += c
    if L > tau:
        R = {o: int(dstart[np.argmax(owner == o)]) for o in range(P) if no[o]}
        for l in range(tau, L):
            for o in range(P):
                if no[o]:
                    segs.append((l * W * 64 + R[o], int(base[P + o]) * 64 + (l - tau) * _wpl(no[o]) * 64,
                                 int(no[o])))
    segs_t = torch.tensor(np.array(segs, dtype=np.int64).reshape(-1, 3), dtype=torch.int64, device=dev)
    src = torch.cat([_i64(p) for p in parts]) if parts else torch.zeros(0, dtype=torch.int64, device=dev)

    # node table: levels < tau from the digit counts (a class of level k is a
    # node when non-empty, starting at C_k(p)); levels >= tau from the owners,
    # in owner order (= ascending digit ranges) within every level
    top_k, top_s, counts = [], [], []
    for k in range(tau):
        w = tau - k
        c = 0
        for p in range(1 << k):
            if D[p << w:(p + 1) << w].sum():
                top_k.append(p)
                top_s.append(int(dstart[p << w]))
                c += 1
        counts.append(c)
    kparts = [torch.tensor(top_k, dtype=torch.int64, device=dev)]
    sparts = [torch.tensor(top_s, dtype=torch.int64, device=dev)]
    if L > tau:
        offs = [np.concatenate(([0], np.cumsum(c))).astype(np.int64) for c in node_cnts]
        for l in range(tau, L):
            c = 0
            for o in range(P):
                a, b = int(offs[o][l - tau]), int(offs[o][l - tau + 1])
                if b > a:
                    kparts.append(node_parts[o][a:b, 0])
                    sparts.append(node_parts[o][a:b, 1])
                    c += b - a
            counts.append(c)
    ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    total = int(ptr[-1])
    t = ops.create(n, sigma, eb, total, dev)
    if W:
        ops.gather_bits(src, segs_t, _i64(t.bits))
    _i64(t.level_node_ptr).copy_(torch.from_numpy(ptr).to(dev))
    if total:
        _i32(t.node_key).copy_(torch.cat(kparts).to(torch.int32))
        _i32(t.node_start).copy_(torch.cat(sparts).to(torch.int32))
    ops.finish(t)
    return t
