"""Check bench.py's reference-arm extrapolation against a full-length reference run (CPU only).

    python tools/ref_extrapolation_check.py N ROWS     (e.g. 32768 4096; needs oracle/_ref)

Prints the extrapolated sparse-attention time of three steps (and the plain covered-pair
ratio) next to the measured wall time of the reference's sparse_attention over all N rows.
"""
import sys, time; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, torch, bench
n=int(sys.argv[1]); R=int(sys.argv[2])
args = bench.parse(["--n", str(n), "--indexer", "random", "--tau-v", "0.3", "--tau-s", "0.6", "--d-h", "256"])
q, k, v, prm, budgets, info = bench.reference_inputs(args)
ref = bench.ReferenceLayer(args, q, k, v, prm, budgets, 8, R)
recs=[ref.step(i) for i in range(3)]
print([ (round(r["attn_est_s"],2), round(r["attn_naive_pair_ratio_s"],2)) for r in recs])
ref.q = q.float().numpy().astype(np.float64)
w, hs = ref._sparse(n)
print("actual wall", w, "makespan of actual per-head", ref._makespan(hs))
