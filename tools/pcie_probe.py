"""Pinned host<->device copy throughput on this box: H2D alone, D2H alone, both at once
(separate streams), at the bench's e2e byte counts. Prints one JSON line."""
import json

import torch

dev = torch.device("cuda", 0)
h2d_b, d2h_b = 1610612736, 1090519040
hi = torch.empty(h2d_b, dtype=torch.uint8).pin_memory()
ho = torch.empty(d2h_b, dtype=torch.uint8).pin_memory()
di = torch.empty(h2d_b, dtype=torch.uint8, device=dev)
do = torch.empty(d2h_b, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timed(lambda: di.copy_(hi, non_blocking=True))
t_d2h = timed(lambda: ho.copy_(do, non_blocking=True))
t_both = timed(both)
print(json.dumps({"h2d_ms": round(t_h2d, 3), "h2d_GBs": round(h2d_b / t_h2d / 1e6, 1),
                  "d2h_ms": round(t_d2h, 3), "d2h_GBs": round(d2h_b / t_d2h / 1e6, 1),
                  "both_ms": round(t_both, 3)}))
