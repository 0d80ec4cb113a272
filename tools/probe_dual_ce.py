"""Do two concurrent D2H copy-engine streams beat one? 256 MiB and 6.55 MB pinned D2H as one copy
vs split in two halves on two streams (and four quarters on four)."""
import json
import torch

N = 256 << 20
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]
main = torch.cuda.current_stream()


def run(nbytes, parts, reps):
    def once():
        ev = torch.cuda.Event()
        ev.record(main)
        for i in range(parts):
            s = ss[i]
            s.wait_event(ev)
            a, b = i * nbytes // parts, (i + 1) * nbytes // parts
            with torch.cuda.stream(s):
                h[a:b].copy_(d[a:b], non_blocking=True)
        for i in range(parts):
            main.wait_stream(ss[i])
    for _ in range(3):
        once()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(main)
    for _ in range(reps):
        once()
    t1.record(main)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / reps
    return nbytes / ms / 1e6


for nbytes, reps in ((N, 10), (6_553_600, 200)):
    for parts in (1, 2, 4):
        print(json.dumps({"bytes": nbytes, "parts": parts, "d2h_gbs": round(run(nbytes, parts, reps), 2)}))
