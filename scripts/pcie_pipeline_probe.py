"""Chunked H2D -> D2H pipeline without kernels, with per-chunk event
timelines (not product code): is the host-buffer step's gap to the
concurrent-copy ceiling in the copies themselves?"""
import torch

n = 25557032
hin = torch.empty(n, pin_memory=True)
hout = torch.empty(n, pin_memory=True)
d = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
M = 1 << 20


def cuts_for(chunk):
    c = [0, M, 3 * M]
    end = n - 3 * M
    m = (end - 3 * M + chunk - 1) // chunk
    for i in range(1, m):
        c.append(3 * M + (end - 3 * M) * i // m // 8192 * 8192)
    c += [end, n - M, n]
    return c


def run(cuts, record=False):
    ev = []
    main = torch.cuda.current_stream()
    s1.wait_stream(main)
    for a, b in zip(cuts[:-1], cuts[1:]):
        e = [torch.cuda.Event(enable_timing=record) for _ in range(4)]
        with torch.cuda.stream(s1):
            e[0].record()
            d[a:b].copy_(hin[a:b], non_blocking=True)
            e[1].record()
        s2.wait_event(e[1])
        with torch.cuda.stream(s2):
            e[2].record()
            hout[a:b].copy_(d[a:b], non_blocking=True)
            e[3].record()
        ev.append(e)
    main.wait_stream(s2)
    return ev


for chunk in (2 * M, 4 * M, 8 * M):
    cuts = cuts_for(chunk)
    run(cuts)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run(cuts)
    b.record()
    torch.cuda.synchronize()
    print(f"chunk {chunk // M} Mi, {len(cuts) - 1} chunks: {a.elapsed_time(b) / 10:.3f} ms per step")
cuts = cuts_for(4 * M)
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
ev = run(cuts, record=True)
torch.cuda.synchronize()
for (a, b), e in zip(zip(cuts[:-1], cuts[1:]), ev):
    mb = (b - a) * 4 / 1e6
    h = (t0.elapsed_time(e[0]), t0.elapsed_time(e[1]))
    dd = (t0.elapsed_time(e[2]), t0.elapsed_time(e[3]))
    print(f"  {mb:6.1f} MB  H2D {h[0]:.3f}-{h[1]:.3f} ({mb / (h[1] - h[0]) / 1e3:.1f} GB/s)  "
          f"D2H {dd[0]:.3f}-{dd[1]:.3f} ({mb / (dd[1] - dd[0]) / 1e3:.1f} GB/s)")
