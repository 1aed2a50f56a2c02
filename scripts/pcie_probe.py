"""PCIe probe on the GPU box: pinned H2D / D2H bandwidth alone and concurrent
(decides how far the host-buffer e2e path can go). Prints one JSON line."""

import json
import time

import torch


def timed(fn, reps=5):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    n = 128 << 20
    h_a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_b = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    res["h2d_GBs"] = n / timed(lambda: d_a.copy_(h_a, non_blocking=True)) / 1e9
    res["d2h_GBs"] = n / timed(lambda: h_b.copy_(d_b, non_blocking=True)) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)
        with torch.cuda.stream(s2):
            h_b.copy_(d_b, non_blocking=True)

    t = timed(both)
    res["concurrent_each_GBs"] = n / t / 1e9
    res["concurrent_total_GBs"] = 2 * n / t / 1e9

    def chunked(k=16):
        c = n // k
        with torch.cuda.stream(s1):
            for i in range(k):
                d_a[i * c:(i + 1) * c].copy_(h_a[i * c:(i + 1) * c], non_blocking=True)
        with torch.cuda.stream(s2):
            for i in range(k):
                h_b[i * c:(i + 1) * c].copy_(d_b[i * c:(i + 1) * c], non_blocking=True)

    t = timed(chunked)
    res["chunked16_concurrent_total_GBs"] = 2 * n / t / 1e9
    # same host buffer both directions (aliasing rows, as step_host in-place)
    def alias():
        c = n // 16
        with torch.cuda.stream(s1):
            for i in range(16):
                d_a[i * c:(i + 1) * c].copy_(h_a[i * c:(i + 1) * c], non_blocking=True)
        with torch.cuda.stream(s2):
            for i in range(16):
                h_a[i * c:(i + 1) * c].copy_(d_b[i * c:(i + 1) * c], non_blocking=True)

    t = timed(alias)
    res["alias16_concurrent_total_GBs"] = 2 * n / t / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
