"""Pinned host <-> device copy bandwidth on the box: H2D alone, D2H alone, both at once
(separate streams) — the ceiling for the host-buffer apply's overlapped transfers."""
import json, time
import torch
n = 650 * 1024 * 1024 // 4
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True); h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float32, device="cuda"); d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3
for _ in range(2): run(True, True, 1)
res = {"bytes": n * 4, "h2d_ms": run(True, False), "d2h_ms": run(False, True), "both_ms": run(True, True)}
res.update({k.replace("_ms", "_GBps"): round(n * 4 / (v * 1e-3) / 1e9 * (2 if k == "both_ms" else 1), 1) for k, v in list(res.items()) if k.endswith("_ms")})
print(json.dumps(res))
