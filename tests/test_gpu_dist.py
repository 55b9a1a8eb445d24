"""GPU checks of the sharded build: the C-ABI helpers
(wt_digit_counts, wt_digits, wt_partition, wt_gather_bits, wt_create /
wt_finish) against plain numpy, and build_sharded with the CUDA ops for P
simulated ranks (threads of one process, tests/dist_helpers.ThreadComm) and
for a real one-rank NCCL group, bit-exact with the oracle's tree of the whole
sequence."""
from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu
KEYS = ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super")


def _cmp(got, want, what=""):
    for k in KEYS:
        assert got[k].shape == want[k].shape, (what, k)
        assert np.array_equal(got[k], want[k]), (what, k)


@pytest.mark.parametrize("dtype,sigma,tau,shift", [(np.uint8, 256, 8, 0), (np.uint16, 3000, 8, 4),
                                                   (np.uint32, 1 << 20, 8, 12), (np.uint32, 1 << 20, 3, 17),
                                                   (np.uint8, 5, 1, 2)])
@pytest.mark.parametrize("n", [0, 1, 4095, 4097, 100003])
def test_partition_and_counts(n, dtype, sigma, tau, shift):
    from paper_1407_8142_b200 import wt
    S = gen.uniform_below(n, sigma, seed=n + tau, dtype=dtype)
    St = torch.from_numpy(S).cuda()
    d = (S.astype(np.int64) >> shift) & ((1 << tau) - 1)
    got = wt.partition(St, shift, tau).cpu().numpy()
    assert np.array_equal(got, S[np.argsort(d, kind="stable")])
    cnt = wt.digit_counts(St, sigma, shift, tau).cpu().numpy()
    assert np.array_equal(cnt, np.bincount(d, minlength=1 << tau))
    dg = wt.digits(St, shift, tau).cpu().numpy()
    assert np.array_equal(dg, d.astype(np.uint8))


def test_digit_counts_validates():
    from paper_1407_8142_b200 import wt
    with pytest.raises(wt.WtError) as e:
        wt.digit_counts(torch.tensor([1, 2, 9], dtype=torch.uint8).cuda(), 4, 0, 2)
    assert e.value.code == wt.WT_ESYMBOL


@pytest.mark.parametrize("seed", range(4))
def test_gather_bits(seed):
    from paper_1407_8142_b200 import wt
    rng = np.random.default_rng(seed)
    src = rng.integers(0, 2**63, size=5000, dtype=np.int64)
    sb = np.unpackbits(src.view(np.uint8), bitorder="little")
    dst_words = 3000 + seed * 1000
    segs, pos = [], int(rng.integers(0, 100))
    while True:
        ln = int(rng.integers(1, 300 if seed % 2 else 5000))
        if pos + ln > dst_words * 64:
            break
        segs.append((pos, int(rng.integers(0, sb.size - ln)), ln))
        pos += ln + int(rng.integers(0, 3) * rng.integers(0, 200))
    want = np.zeros(dst_words * 64, dtype=np.uint8)
    for d, s, ln in segs:
        want[d:d + ln] = sb[s:s + ln]
    dst = torch.full((dst_words,), -1, dtype=torch.int64, device="cuda")
    wt.gather_bits(torch.from_numpy(src).cuda(), torch.tensor(segs, dtype=torch.int64).cuda(), dst)
    assert np.array_equal(np.unpackbits(dst.cpu().numpy().view(np.uint8), bitorder="little"), want)


def _sharded_threads(S, sigma, cuts):
    from paper_1407_8142_b200 import dist as wdist
    from tests.dist_helpers import LockedOps, ThreadComm, host_arrays
    P = len(cuts) - 1
    comms = ThreadComm.group(P)
    lock = threading.Lock()
    res, errs = [None] * P, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            St = torch.from_numpy(S[cuts[r]:cuts[r + 1]].copy()).cuda()
            t = wdist.build_sharded(St, sigma, comms[r], LockedOps(wdist.CudaOps(), lock))
            res[r] = host_arrays(t)
            t.free()
        except Exception as e:  # pragma: no cover
            import traceback
            errs.append(traceback.format_exc())
            comms[r].sh.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errs, errs[0]
    return res


@pytest.mark.parametrize("n,sigma,dtype,P", [
    (200000, 1 << 16, np.uint32, 4), (100000, 1000, np.uint16, 3), (150000, 256, np.uint8, 2),
    (50000, 4, np.uint8, 3), (120000, 1 << 24, np.uint32, 5), (30000, 1 << 32, np.uint32, 2),
    (0, 100, np.uint8, 2)])
def test_sharded_threads(n, sigma, dtype, P):
    S = gen.uniform_below(n, sigma, seed=7 + P, dtype=dtype)
    rng = np.random.default_rng(P)
    cuts = np.sort(np.concatenate(([0, n], rng.integers(0, n + 1, P - 1)))).astype(np.int64)
    want = oracle.build(S, sigma)
    for r, got in enumerate(_sharded_threads(S, sigma, cuts)):
        _cmp(got, want, f"rank {r}")


def test_sharded_threads_config3():
    cfg = gen.CONFIGS[3]
    S = gen.config_input(cfg, 1 << 22)
    cuts = np.array([0, 1 << 20, 3 << 20, 1 << 22])
    want = oracle.build(S, cfg.sigma)
    for got in _sharded_threads(S, cfg.sigma, cuts):
        _cmp(got, want)


@pytest.mark.parametrize("exchange", [False, True])
def test_sharded_nccl_one_rank(exchange):
    import torch.distributed as dist
    from paper_1407_8142_b200 import dist as wdist
    from tests.dist_helpers import host_arrays
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        S = gen.uniform_below(300000, 1 << 16, seed=3, dtype=np.uint32)
        # exchange=True: digit counts, top levels, all_to_all_single and the
        # all-gathers of assemble() all go through NCCL (world size 1)
        t = wdist.build_sharded(torch.from_numpy(S).cuda(), 1 << 16, exchange=exchange)
        _cmp(host_arrays(t), oracle.build(S, 1 << 16))
        t.free()
    finally:
        dist.destroy_process_group()
