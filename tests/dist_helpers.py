"""Test infrastructure for the sharded build (paper_1407_8142_b200/dist.py).

* ``HostOps``: the local steps of the sharded build on CPU tensors -- the
  chunk builds come from the CPU oracle, the digit counting / partition /
  bit gather are written out in numpy.  It lets the gloo tests check the
  orchestration (collectives, owners, offsets, run placement, node tables)
  on CPU; the CUDA steps themselves are checked on the GPU
  (tests/test_gpu_dist.py).
* ``ThreadComm``: the collectives of ``TorchComm`` for P ranks simulated by P
  threads of one process (host barriers only, no kernel ever waits on
  another rank's kernel), so the CUDA path can run with P > 1 on one GPU.
"""
from __future__ import annotations

import threading

import numpy as np
import torch

import oracle
from tests import pins


class _HostTree:
    def __init__(self, **kw):
        self.__dict__.update(kw)


class HostOps:
    def digit_counts(self, S, sigma, shift, tau):
        from paper_1407_8142_b200.wt import WtError, WT_ESYMBOL
        a = S.numpy().astype(np.int64)
        if a.size and int(a.max()) >= sigma:
            raise WtError(WT_ESYMBOL, "digit_counts")
        return torch.from_numpy(np.bincount((a >> shift) & ((1 << tau) - 1), minlength=1 << tau).astype(np.int64))

    def digits(self, S, shift, tau):
        return torch.from_numpy(((S.numpy().astype(np.int64) >> shift) & ((1 << tau) - 1)).astype(np.uint8))

    def partition(self, S, shift, tau):
        a = S.numpy()
        d = (a.astype(np.int64) >> shift) & ((1 << tau) - 1)
        return torch.from_numpy(a[np.argsort(d, kind="stable")].copy())

    def build(self, S, sigma):
        o = oracle.build(S.numpy(), sigma)
        return _HostTree(bits=torch.from_numpy(o["bits"].view(np.int64)),
                         level_node_ptr=torch.from_numpy(o["level_node_ptr"].view(np.int64)),
                         node_key=torch.from_numpy(o["node_key"].view(np.int32)),
                         node_start=torch.from_numpy(o["node_start"].view(np.int32)))

    def create(self, n, sigma, eb, total, device):
        L = (int(sigma) - 1).bit_length()
        W = ((n + 511) // 512) * 8
        return _HostTree(n=n, sigma=sigma, levels=L, bits=torch.zeros(L * W, dtype=torch.int64),
                         level_node_ptr=torch.zeros(L + 1, dtype=torch.int64),
                         node_key=torch.zeros(total, dtype=torch.int32),
                         node_start=torch.zeros(total, dtype=torch.int32))

    def gather_bits(self, src, segs, dst):
        sb = np.unpackbits(src.numpy().view(np.uint8), bitorder="little")
        out = np.zeros(dst.numel() * 64, dtype=np.uint8)
        for d, s, ln in segs.numpy().reshape(-1, 3):
            out[d:d + ln] = sb[s:s + ln]
        dst.copy_(torch.from_numpy(np.packbits(out, bitorder="little").view(np.int64)))

    def finish(self, t):
        blk, sup = pins.rank_directory_bruteforce(t.bits.numpy().view(np.uint64), t.n, t.levels)
        t.rank_block, t.rank_super = torch.from_numpy(blk), torch.from_numpy(sup)


def host_arrays(t) -> dict:
    """The §8(b) arrays of a tree built with HostOps or the CUDA ops."""
    g = lambda x: x.cpu().numpy()  # noqa: E731
    return {"bits": g(t.bits).view(np.uint64), "level_node_ptr": g(t.level_node_ptr).view(np.uint64),
            "node_key": g(t.node_key).view(np.uint32), "node_start": g(t.node_start).view(np.uint32),
            "rank_block": g(t.rank_block).view(np.uint16), "rank_super": g(t.rank_super).view(np.uint64)}


class ThreadComm:
    """P ranks as P threads: collectives exchange tensor references at a barrier."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank):
        self.sh, self.rank, self.world = shared, rank, shared.world

    @classmethod
    def group(cls, world):
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def _exchange(self, obj, take):
        """Publish obj, then copy what this rank needs (take) before anyone
        may release its buffers (like a real collective, which copies)."""
        self.sh.barrier.wait()
        self.sh.slots[self.rank] = obj
        self.sh.barrier.wait()
        out = take(list(self.sh.slots))
        torch.cuda.synchronize()
        self.sh.barrier.wait()
        return out

    def all_gather(self, t):
        return self._exchange(t, lambda xs: [x.clone() for x in xs])

    def all_gather_v(self, t):
        return self._exchange(t, lambda xs: [x.clone() for x in xs])

    def all_to_all_v(self, t, send_counts):
        offs = np.concatenate(([0], np.cumsum(send_counts))).astype(np.int64)
        return self._exchange([t[offs[j]:offs[j + 1]] for j in range(self.world)],
                              lambda ps: torch.cat([ps[j][self.rank] for j in range(self.world)]).clone())


class LockedOps:
    """Serialise the library calls of simulated ranks (one process, one GPU)."""

    def __init__(self, ops, lock):
        self.ops, self.lock = ops, lock

    def __getattr__(self, name):
        f = getattr(self.ops, name)

        def call(*a, **k):
            with self.lock:
                r = f(*a, **k)
                torch.cuda.synchronize()
                return r
        return call
