import sys, time, torch, json
sys.path.insert(0, ".")
def run(streams, nbytes=8 << 30, reps=3, chunk=512 << 20):
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    ss = [torch.cuda.Stream() for _ in range(streams)]
    best = 0
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for i, a in enumerate(range(0, nbytes, chunk)):
            with torch.cuda.stream(ss[i % streams]):
                h[a:a + chunk].copy_(d[a:a + chunk], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
    return best
for s in (1, 2, 3, 4):
    print(json.dumps({"d2h_streams": s, "GBs": round(run(s), 2)}), flush=True)
