"""Builds issued concurrently from several host threads, each on its own CUDA
stream (the library keeps no per-call state in shared host buffers): every
tree, matrix and Huffman-shaped tree is bit-exact with the oracle."""
from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu


def test_concurrent_builds():
    import paper_1407_8142_b200 as wt
    inputs = [(gen.uniform_below(200000 + 1000 * i, s, seed=i, dtype=np.uint32), s)
              for i, s in enumerate([1 << 16, 1000, 1 << 20, 256, 3, 1 << 32])]
    want = [oracle.build(S, s) for S, s in inputs]
    want_wm = [oracle.wm_build(S, s) for S, s in inputs[:3]]
    errors = []

    def run(i):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            S, s = inputs[i]
            with torch.cuda.stream(st):
                St = torch.from_numpy(S).cuda()
                for _ in range(3):
                    t = wt.build(St, s, stream=st)
                    got = t.numpy()
                    for k in ("bits", "level_node_ptr", "node_key", "node_start", "rank_block", "rank_super"):
                        if not np.array_equal(got[k], want[i][k]):
                            errors.append((i, k))
                    assert t.total_nodes == want[i]["total_nodes"]
                    t.free()
                    if i < 3:
                        m = wt.wm_build(St, s, stream=st)
                        g = m.numpy()
                        for k in ("bits", "zeros", "rank_block", "rank_super"):
                            if not np.array_equal(g[k], want_wm[i][k]):
                                errors.append((i, "wm_" + k))
                        m.free()
        except Exception as e:  # pragma: no cover
            errors.append((i, repr(e)))

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(inputs))]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errors, errors[:5]


def test_free_waits_for_query_streams():
    """wt_free / wm_free release memory only after the queries enqueued on
    other streams (select index built on a side stream, long query batches):
    results stay correct while the freed memory is immediately reused."""
    import paper_1407_8142_b200 as wt
    S = gen.uniform_below(1 << 20, 1 << 16, seed=11, dtype=np.uint32)
    St = torch.from_numpy(S).cuda()
    pos = torch.randint(0, S.size, (1 << 22,), device="cuda", dtype=torch.int64)
    want = torch.from_numpy(S.astype(np.int64)).cuda()[pos]
    for build in (wt.build, wt.wm_build):
        side = torch.cuda.Stream()
        t = build(St, 1 << 16)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            t.select_index(stream=side)
            got = t.access(pos, stream=side)
        t.free()  # enqueued on the build stream; must wait for `side`
        junk = [torch.full((1 << 24,), 0x55, dtype=torch.uint8, device="cuda") for _ in range(8)]  # reuse
        torch.cuda.synchronize()
        assert torch.equal(got.to(torch.int64), want)
        del junk


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_devices_one_process():
    """Per-device launch state: builds on cuda:0 then cuda:1 in one process."""
    import paper_1407_8142_b200 as wt
    S = gen.uniform_below(300000, 1 << 16, seed=12, dtype=np.uint32)
    want = oracle.build(S, 1 << 16)
    for d in (0, 1, 0):
        with torch.cuda.device(d):
            t = wt.build(torch.from_numpy(S).cuda(d), 1 << 16)
            got = t.numpy()
            for k in ("bits", "node_key", "rank_block", "rank_super"):
                assert np.array_equal(got[k], want[k]), (d, k)
            t.free()
