"""PCIe copy probe: pinned H2D, D2H and both directions concurrently (1 GPU)."""
import json
import torch

n = 2 << 30  # 2 GiB per buffer
dev = torch.device("cuda:0")
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device=dev)
d_b = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
t_both = timed(both)
print(json.dumps({"bytes": n, "h2d_gbs": n / t_h2d / 1e9, "d2h_gbs": n / t_d2h / 1e9,
                  "both_each_gbs": n / t_both / 1e9, "both_total_gbs": 2 * n / t_both / 1e9}))
