"""Raw pinned H2D / D2H bandwidth on the box (one or two copy streams, chunked),
to bound the e2e numbers (experiments)."""
import json, torch
dev = torch.device("cuda", 0)
MB = 1 << 20
out = {}
for size_mb in (54, 216):
    h = torch.empty(size_mb * MB, dtype=torch.uint8).pin_memory()
    d = torch.empty(size_mb * MB, dtype=torch.uint8, device=dev)
    for nstreams in (1, 2, 4):
        ss = [torch.cuda.Stream(dev) for _ in range(nstreams)]
        chunk = size_mb * MB // nstreams
        for _ in range(3):
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for s in ss:
            s.wait_event(e0)
        for _ in range(reps):
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in ss:
            ev = torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        out[f"h2d_{size_mb}MB_{nstreams}s_GBs"] = round(reps * size_mb * MB / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)
    # D2H and bidirectional
    h2 = torch.empty(size_mb * MB, dtype=torch.uint8).pin_memory()
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s1.wait_event(e0); s2.wait_event(e0)
    for _ in range(10):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d, non_blocking=True)
    for s in (s1, s2):
        ev = torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
    e1.record(); torch.cuda.synchronize()
    out[f"bidir_{size_mb}MB_each_GBs"] = round(10 * size_mb * MB / (e0.elapsed_time(e1) / 1e3) / 1e9, 1)
print(json.dumps(out))
