"""D2H throughput of the cfg3 output size (2.4 GB) into pinned host memory: one copy vs the same
bytes split across 2 / 4 streams (copy engines), CUDA events, best of 3."""
import json, torch
n = 2415919104
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
res = {}
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step = n // parts
        for i, s in enumerate(streams):
            s.wait_event(a)
            with torch.cuda.stream(s):
                host[i * step:(i + 1) * step].copy_(dev[i * step:(i + 1) * step], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    res[f"d2h_{parts}_streams_gbs"] = n / best / 1e6
hin = torch.empty(16777216, dtype=torch.uint8, pin_memory=True)
print(json.dumps(res))
