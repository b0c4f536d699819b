"""Generate tests/golden/reference_vectors.json FROM THE REFERENCE ITSELF.

Runs the unmodified reference library (oracle/_ref/libvspref.so, compiled from
/root/reference/proj/include by oracle/Makefile) on small seeded inputs and records inputs
and outputs. The fixtures pin the C restatement (oracle/vsp_oracle.c) and the GPU parity
tests on machines where /root/reference is absent (the GPU box). Re-run here with:

    make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    ref = oracle.ref()
    rng = np.random.default_rng(20260304)
    out = {"source": "reference vsp:: functions via oracle/_ref (ref_shim.cpp)", "cases": {}}
    C = out["cases"]

    # merge_row_columns (merge.hpp:18-56): hand cases + random
    merges = [([0, 5], [0, 2], 4), ([], [0], 7), ([1, 9], [], 3), ([2], [3], 5), ([], [], 4)]
    for _ in range(40):
        n = int(rng.integers(1, 60))
        iv = sorted(rng.choice(n, size=int(rng.integers(0, n + 1)), replace=False).tolist())
        is_ = sorted(rng.choice(n, size=int(rng.integers(0, n + 1)), replace=False).tolist())
        merges.append((iv, is_, int(rng.integers(0, n))))
    C["merge_row_columns"] = [dict(iv=a, is_=b, i=i, out=ref.merge_row_columns(a, b, i).tolist())
                              for a, b, i in merges]

    # merge_path_partition (merge.hpp:69-95)
    mp = [([1, 3, 5], [2, 4, 6], 2)]
    for _ in range(20):
        a = sorted(rng.integers(0, 50, size=int(rng.integers(0, 20))).tolist())
        b = sorted(rng.integers(0, 50, size=int(rng.integers(0, 20))).tolist())
        mp.append((a, b, int(rng.integers(1, 8))))
    C["merge_path_partition"] = [dict(a=a, b=b, p=p, cuts=[list(map(int, c)) for c in ref.merge_path_partition(a, b, p)])
                                 for a, b, p in mp]

    # cumulative_budget (sparsity.hpp:51-79)
    cb = []
    s = [0.5, 0.25, 0.125, 0.125]
    for tau in (0.5, 0.6, 0.75, 0.76, 0.875, 0.9, 1.0):
        cb.append(dict(scores=s, tau=tau, min=1, max=-1, k=ref.cumulative_budget(s, tau)))
    for mn, mx, tau in ((3, -1, 0.5), (10, -1, 0.5), (1, 2, 1.0), (1, 100, 1.0)):
        cb.append(dict(scores=s, tau=tau, min=mn, max=mx, k=ref.cumulative_budget(s, tau, min_budget=mn, max_budget=mx)))
    for _ in range(30):
        n = int(rng.integers(1, 200))
        p = rng.exponential(size=n)
        p = (p / p.sum()).tolist()
        tau = float(1e-3 + 0.999 * rng.random())
        cb.append(dict(scores=p, tau=tau, min=1, max=-1, k=ref.cumulative_budget(p, tau)))
    C["cumulative_budget"] = cb

    # topk_indices (sparsity.hpp:83-97), quantized for ties
    tk = [dict(scores=[0.2, 0.5, 0.2, 0.1], k=k) for k in (1, 2, 3, 4)]
    tk += [dict(scores=[0.3, 0.2, 0.2, 0.3], k=k) for k in (2, 3)]
    tk += [dict(scores=[0.4, 0.1, 0.1, 0.4], k=2), dict(scores=[0.1, 0.4, 0.4, 0.1], k=2)]
    for _ in range(40):
        n = int(rng.integers(1, 80))
        sc = (rng.integers(0, 8, size=n) / 8.0).tolist()
        tk.append(dict(scores=sc, k=int(rng.integers(1, n + 1))))
    for t in tk:
        t["out"] = ref.topk_indices(t["scores"], t["k"]).tolist()
    C["topk_indices"] = tk

    # select_pattern (sparsity.hpp:105-114)
    sp = [dict(sv=[1 / 8] * 8, ss=[1 / 8] * 8, tau_v=0.5, tau_s=0.25, min=1, max=-1),
          dict(sv=[0.0, 0.0, 1.0, 0.0], ss=[0.0, 0.0, 0.0, 1.0], tau_v=0.9, tau_s=0.9, min=1, max=-1)]
    for _ in range(20):
        n = int(rng.integers(2, 300))
        a = rng.exponential(size=n) ** 3
        b = rng.exponential(size=n) ** 3
        sp.append(dict(sv=(a / a.sum()).tolist(), ss=(b / b.sum()).tolist(), tau_v=float(rng.uniform(0.05, 1.0)),
                       tau_s=float(rng.uniform(0.05, 1.0)), min=int(rng.integers(1, 4)),
                       max=int(rng.choice([-1, int(rng.integers(4, 50))]))))
    for c in sp:
        iv, is_ = ref.select_pattern(c["sv"], c["ss"], c["tau_v"], c["tau_s"], c["min"], c["max"])
        c["i_v"], c["i_s"] = iv.tolist(), is_.tolist()
    C["select_pattern"] = sp

    # indexer_forward (indexer.hpp:77-120), both mappings
    ix = []
    for rev in (True, False):
        n, d, dh = 11, 4, 6
        k = rng.standard_normal((n, d))
        v = rng.standard_normal((n, d))
        p = dict(w_u=(rng.uniform(-1, 1, size=(2 * d, dh)) / np.sqrt(2 * d)), b_u=0.3 * rng.standard_normal(dh),
                 w_v=rng.standard_normal(dh), b_v=0.1, w_s=rng.standard_normal(dh), b_s=-0.2)
        r = ref.indexer_forward(k, v, p, reverse=rev)
        ix.append(dict(reverse=rev, k=k.tolist(), v=v.tolist(), **{a: (b.tolist() if hasattr(b, "tolist") else b)
                                                                   for a, b in p.items()},
                       **{a: b.tolist() for a, b in r.items()}))
    C["indexer_forward"] = ix

    # attention: blockwise (attention.hpp:96-145) and sparse (150-194)
    at = []
    for n, d, block in ((20, 8, 7), (33, 16, 32), (5, 4, 1)):
        q, k, v = (rng.standard_normal((n, d)) for _ in range(3))
        iv = sorted(rng.choice(n, size=n // 4, replace=False).tolist())
        is_ = sorted(set(rng.choice(n, size=n // 3, replace=False).tolist()) | {0})
        at.append(dict(q=q.tolist(), k=k.tolist(), v=v.tolist(), block=block, i_v=iv, i_s=is_,
                       dense=ref.blockwise_attention(q, k, v, block=block).tolist(),
                       sparse=ref.sparse_attention(q, k, v, iv, is_, block=block).tolist()))
    C["attention"] = at

    # aggregate_streaming (vsaggregate.hpp:62-127)
    ag = []
    for n, d, block in ((17, 8, 4), (40, 16, 64)):
        q, k = rng.standard_normal((n, d)), rng.standard_normal((n, d))
        vert, sl = ref.aggregate_streaming(q, k, block=block)
        ag.append(dict(q=q.tolist(), k=k.tolist(), block=block, vertical=vert.tolist(), slash=sl.tolist()))
    C["aggregate_streaming"] = ag

    # apply_rope (rope.hpp:63-79): row-index positions, explicit long-context positions, bases
    rp = []
    for n, d, base, positions in ((6, 8, 10000.0, None), (7, 128, 10000.0, [0, 1, 4095, 32768, 65537, 100000, 131071]),
                                  (5, 128, 500000.0, [131071, 3, 77777, 12, 0]), (3, 2, 10000.0, None)):
        x = rng.standard_normal((n, d))
        rp.append(dict(x=x.tolist(), positions=positions, base=base,
                       out=ref.apply_rope(x, positions, base).tolist()))
    C["apply_rope"] = rp

    # distillation: indexer_backward_loss (indexer.hpp:265-272), optimizer_step (:347-363),
    # learning_rate (:322-329)
    ib = []
    for n, d, dh, rev in ((9, 4, 6, True), (13, 8, 16, False), (1, 2, 3, True)):
        k, v = rng.standard_normal((n, d)), rng.standard_normal((n, d))
        pr = {"w_u": rng.uniform(-0.3, 0.3, (2 * d, dh)), "b_u": rng.standard_normal(dh) * 0.1,
              "w_v": rng.standard_normal(dh), "b_v": 0.2, "w_s": rng.standard_normal(dh), "b_s": -0.1}
        tv, ts = rng.random(n), rng.random(n)
        tv, ts = tv / tv.sum(), ts / ts.sum()
        loss, g = ref.indexer_backward(k, v, pr, tv, ts, reverse=rev)
        ib.append(dict(k=k.tolist(), v=v.tolist(), params={x: (y.tolist() if hasattr(y, "tolist") else y)
                                                           for x, y in pr.items()},
                       target_v=tv.tolist(), target_s=ts.tolist(), reverse=rev, loss=loss,
                       grads={x: (y.tolist() if hasattr(y, "tolist") else y) for x, y in g.items()}))
    C["indexer_backward"] = ib
    d, dh = 2, 3
    cnt = 2 * d * dh + 3 * dh + 2
    p0, g0 = rng.standard_normal(cnt), rng.standard_normal(cnt)
    m0, v0 = rng.standard_normal(cnt) * 0.1, rng.random(cnt) * 0.1
    os_ = []
    for step, steps, warmup in ((0, 10, 3), (5, 10, 3), (9, 10, 0)):
        p1, m1, v1 = p0.copy(), m0.copy(), v0.copy()
        oracle.ref_optimizer_step(d, dh, p1, g0, m1, v1, step, steps, warmup, 1e-3)
        os_.append(dict(d=d, d_h=dh, p=p0.tolist(), g=g0.tolist(), m=m0.tolist(), v=v0.tolist(), step=step,
                        steps=steps, warmup=warmup, lr_peak=1e-3,
                        lr=oracle.ref_learning_rate(step, steps, warmup, 1e-3),
                        p_out=p1.tolist(), m_out=m1.tolist(), v_out=v1.tolist()))
    C["optimizer_step"] = os_

    path = os.path.join(HERE, "reference_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
