"""Pinned host <-> device copy bandwidth (the e2e ceiling): H2D, D2H, and both at once."""
import json
import torch

n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
bd = timed(both)
print(json.dumps({"h2d_gbs": n / h2d / 1e6, "d2h_gbs": n / d2h / 1e6, "bidir_each_gbs": n / bd / 1e6,
                  "bidir_ms_for_1GiB_each_way": bd}))
