"""Host logic of the sharded build on CPU: world sizes 1
(every exchange collective forced), 2 and 3 over gloo (torch.distributed, 127.0.0.1), the local steps done by
tests/dist_helpers.HostOps (oracle chunk builds + numpy), the result compared
array by array with the oracle's tree of the whole sequence."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [  # (n, sigma, dtype, chunk fractions)
    (3000, 4, "uint8", (0.5, 0.5)),            # L <= tau: no exchange
    (5000, 256, "uint8", (0.3, 0.7)),          # L == tau
    (6000, 1000, "uint16", (0.5, 0.5)),        # L = 10: exchange of 2-bit tails
    (9000, 1 << 16, "uint32", (0.2, 0.8)),     # L = 16
    (4000, 3000, "uint16", (0.0, 1.0)),        # an empty chunk
    (2500, 1 << 20, "uint32", (0.6, 0.4)),     # L = 20
    (0, 77, "uint8", (0.5, 0.5)),              # n = 0
    (100, 1, "uint8", (0.5, 0.5)),             # sigma = 1
]


def _seq(n, sigma, dtype, seed):
    import gen
    return gen.uniform_below(n, sigma, seed=seed, dtype=np.dtype(dtype).type)


def _worker(rank, world, port, q, cases):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1407_8142_b200 import dist as wdist
    from tests.dist_helpers import HostOps, host_arrays
    out = []
    try:
        for ci, (n, sigma, dtype, fr) in enumerate(cases):
            S = _seq(n, sigma, dtype, 100 + ci)
            cuts = np.concatenate(([0], np.cumsum(np.array(fr) * n).astype(np.int64)))
            cuts[-1] = n
            if world == 3:
                cuts = np.array([0, n // 5, n // 2, n])
            if world == 1:
                cuts = np.array([0, n])
            lo, hi = int(cuts[rank]), int(cuts[rank + 1])
            # exchange=True: world size 1 still runs every exchange collective
            t = wdist.build_sharded(torch.from_numpy(S[lo:hi].copy()), sigma, wdist.TorchComm(), HostOps(),
                                    exchange=True)
            out.append(host_arrays(t))
            # distributed output: the same parts assembled on demand give the same tree
            part = wdist.build_sharded(torch.from_numpy(S[lo:hi].copy()), sigma, wdist.TorchComm(), HostOps(),
                                       gather=False, exchange=True)
            if isinstance(part, wdist.ShardedPart):
                # this rank's top-level runs: lengths are its class counts, offsets inside the level
                for k in range(part.tau):
                    for p_, (off, ln) in part.place_top(k).items():
                        assert 0 <= off and off + ln <= n
                t2 = wdist.assemble(part, wdist.TorchComm(), HostOps())
                out[-1] = (out[-1], host_arrays(t2))
            else:
                out[-1] = (out[-1], host_arrays(part))
        # invalid symbol on one rank only: every rank must raise
        bad = np.array([1, 2, 3] if rank == 0 and world > 1 else [1, 9, 2], dtype=np.uint8)
        try:
            wdist.build_sharded(torch.from_numpy(bad), 4, wdist.TorchComm(), HostOps(), exchange=True)
            out.append("no error")
        except Exception as e:  # WtError(WT_ESYMBOL)
            out.append(getattr(e, "code", repr(e)))
        q.put((rank, out))
    except Exception as e:  # pragma: no cover - reported by the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_build_gloo(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, CASES)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank in range(world):
        assert not isinstance(res[rank], str), res[rank]
    for ci, (n, sigma, dtype, _) in enumerate(CASES):
        want = oracle.build(_seq(n, sigma, dtype, 100 + ci), sigma)
        for rank in range(world):
            for got in res[rank][ci]:  # gathered build, distributed parts assembled
                for k in ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super"):
                    assert np.array_equal(got[k], want[k]), (ci, rank, k)
    for rank in range(world):
        assert res[rank][-1] == -2  # WT_ESYMBOL on every rank


def test_plan_owners():
    from paper_1407_8142_b200.dist import plan_owners
    D = np.array([5, 0, 0, 10, 1, 4], dtype=np.int64)
    o = plan_owners(D, 3)
    assert list(o) == sorted(o) and o[0] == 0 and o.max() <= 2
    assert list(plan_owners(np.zeros(4, np.int64), 2)) == [0, 0, 0, 0]
