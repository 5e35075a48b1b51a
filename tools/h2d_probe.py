"""Pinned H2D bandwidth vs number of concurrent copy streams and chunk size
(development aid)."""
import torch

dev = torch.device("cuda", 0)
total = 1 << 30
host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
host.fill_(1)
d = torch.empty(total, dtype=torch.uint8, device=dev)
for nstreams in (1, 2, 4):
    for chunk in (8 << 20, 64 << 20, 256 << 20):
        ss = [torch.cuda.Stream() for _ in range(nstreams)]
        for rep in range(2):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for s in ss:
                s.wait_event(a)
            for i, off in enumerate(range(0, total, chunk)):
                s = ss[i % nstreams]
                with torch.cuda.stream(s):
                    d[off:off + chunk].copy_(host[off:off + chunk], non_blocking=True)
            for s in ss:
                ev = torch.cuda.Event()
                ev.record(s)
                torch.cuda.current_stream().wait_event(ev)
            b.record()
            torch.cuda.synchronize()
        print(f"streams {nstreams} chunk {chunk >> 20:4d} MiB: {total / a.elapsed_time(b) / 1e6:.2f} GB/s", flush=True)
