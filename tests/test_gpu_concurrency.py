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
