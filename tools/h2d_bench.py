"""Pinned host -> HBM copy bandwidth with the expert-sized transfer split over
1..4 concurrent streams (does a second copy engine raise the PCIe rate?)."""
import torch

N = 71651328  # one C2 expert
src = torch.empty(N * 4, dtype=torch.uint8).pin_memory()
dst = torch.empty(N * 4, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 3, 4):
    best = 0.0
    for rep in range(5):
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for s in streams[:ns]:
            s.wait_event(ev0)
        per = (N + ns - 1) // ns
        for i, s in enumerate(streams[:ns]):
            with torch.cuda.stream(s):
                a, b = i * per, min(N, (i + 1) * per)
                dst[a:b].copy_(src[a:b], non_blocking=True)
        for s in streams[:ns]:
            ev1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
        ev1.record()
        torch.cuda.synchronize()
        gbs = N / (ev0.elapsed_time(ev1) * 1e-3) / 1e9
        best = max(best, gbs)
    print(f"streams={ns}: best {best:.2f} GB/s for {N/1e6:.1f} MB")
# 4 experts back to back on one stream vs two
for ns in (1, 2):
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for s in streams[:ns]:
        s.wait_event(ev0)
    for k in range(4):
        s = streams[k % ns]
        with torch.cuda.stream(s):
            dst[k * N:(k + 1) * N].copy_(src[k * N:(k + 1) * N], non_blocking=True)
    for s in streams[:ns]:
        torch.cuda.current_stream().wait_stream(s)
    ev1.record()
    torch.cuda.synchronize()
    print(f"4 experts on {ns} stream(s): {4 * N / (ev0.elapsed_time(ev1) * 1e-3) / 1e9:.2f} GB/s")
