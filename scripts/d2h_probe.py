"""Host-link D2H bandwidth under the shapes the pipelined e2e uses: one 256 MiB copy, 8 x 53.7 MB
(one cfg4 build each) into consecutive slices of one pinned buffer, the same split into 6 copies
per build, and both while host processes stream memory (as the host analysis does)."""
import multiprocessing as mp
import os, sys, time
import numpy as np
import torch


def burn(stop):
    a = np.ones(64 << 20, np.uint8)
    b = np.empty_like(a)
    while not stop.is_set():
        np.copyto(b, a)


def run(tag, parts):
    dev = torch.device("cuda", 0)
    d = torch.empty(8 * 53_710_752, dtype=torch.uint8, device=dev)
    h = torch.empty(8 * 53_710_752, dtype=torch.uint8, pin_memory=True)
    s = torch.cuda.Stream(dev)
    best = 1e9
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            off = 0
            for p in parts:
                h[off:off + p].copy_(d[off:off + p], non_blocking=True)
                off += p
            b.record(s)
        s.synchronize()
        best = min(best, a.elapsed_time(b))
    tot = sum(parts)
    print(f"{tag}: {tot / 1e6:.1f} MB in {best:.3f} ms = {tot / best / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__" and "--sweep" not in sys.argv:
    one = [256 << 20]
    builds = [53_710_752] * 8
    six = []
    for _ in range(8):
        six += [658_944 * 3 // 3] * 3 + [17_686_528] * 3
    for load in (0, 8, 15):
        stop = mp.Event()
        ps = [mp.Process(target=burn, args=(stop,)) for _ in range(load)]
        for p in ps:
            p.start()
        time.sleep(0.5)
        run(f"load {load:2d} one 256MiB", one)
        run(f"load {load:2d} 8 builds", builds)
        run(f"load {load:2d} 8 builds x 6 copies", six)
        stop.set()
        for p in ps:
            p.join()


def sweep_pattern():
    """The one-shot cfg5 sweep's copies: 24 chunks, per chunk 3 node tensors (~0.23 MB) and 3 edge
    tensors (~5.6 MB) into six big pinned arrays, plus the same bytes as one copy per chunk."""
    dev = torch.device("cuda", 0)
    nn, ne, K = 29_000, 706_000, 24
    dsrc = [torch.empty((nn if k < 3 else ne) * 8, dtype=torch.uint8, device=dev) for k in range(6)]
    big = [torch.empty(K * (nn if k < 3 else ne) * 8, dtype=torch.uint8, pin_memory=True) for k in range(6)]
    one = torch.empty(K * (3 * nn + 3 * ne) * 8, dtype=torch.uint8, pin_memory=True)
    dall = torch.empty((3 * nn + 3 * ne) * 8, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    for tag in ("6 copies per chunk", "1 copy per chunk", "3 edge copies per chunk"):
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                a.record(s)
                for c in range(K):
                    if tag.startswith("6"):
                        for k in range(6):
                            n = dsrc[k].numel()
                            big[k][c * n:(c + 1) * n].copy_(dsrc[k], non_blocking=True)
                    elif tag.startswith("3"):
                        for k in range(3, 6):
                            n = dsrc[k].numel()
                            big[k][c * n:(c + 1) * n].copy_(dsrc[k], non_blocking=True)
                    else:
                        n = dall.numel()
                        one[c * n:(c + 1) * n].copy_(dall, non_blocking=True)
                b.record(s)
            s.synchronize()
            best = min(best, a.elapsed_time(b))
        tot = K * (3 * ne * 8 + (0 if tag.startswith("3") else 3 * nn * 8))
        print(f"sweep pattern, {tag}: {tot / 1e6:.1f} MB in {best:.3f} ms = {tot / best / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__" and "--sweep" in sys.argv:
    sweep_pattern()
