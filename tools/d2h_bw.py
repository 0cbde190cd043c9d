#!/usr/bin/env python3
"""Pinned D2H / H2D bandwidth on the box (what bounds the dense e2e number): one stream vs
several concurrent copy streams over the same total bytes.

  python tools/d2h_bw.py [--mb 530]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=530)
    a = ap.parse_args()
    nbytes = a.mb << 20
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    for direction in ("d2h", "h2d"):
        for nstreams in (1, 2, 4):
            streams = [torch.cuda.Stream() for _ in range(nstreams)]
            chunk = nbytes // nstreams
            best = 0.0
            for _ in range(5):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for k, s in enumerate(streams):
                    s.wait_event(e0)
                    with torch.cuda.stream(s):
                        if direction == "d2h":
                            host[k * chunk:(k + 1) * chunk].copy_(dev[k * chunk:(k + 1) * chunk], non_blocking=True)
                        else:
                            dev[k * chunk:(k + 1) * chunk].copy_(host[k * chunk:(k + 1) * chunk], non_blocking=True)
                for s in streams:
                    e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
                torch.cuda.current_stream().wait_stream(streams[-1])
                for s in streams:
                    torch.cuda.current_stream().wait_stream(s)
                e1.record()
                torch.cuda.synchronize()
                best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
            print(json.dumps({"dir": direction, "streams": nstreams, "MB": a.mb, "GB_per_s": round(best, 2)}))


if __name__ == "__main__":
    main()
