"""Practical HBM ceiling for small streaming kernels (calibration, not the bench).

    python tools/membench.py

Times a hand-written 256-bit read/write kernel (tools/membench.cu) moving the
same read/write byte mix as each config, through CUDA graphs over rotating
buffers (> 3x L2), with and without programmatic dependent launch (PDL).
"""
import ctypes
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2510_07843_b200 import synth  # noqa: E402

SRC = os.path.join(ROOT, "tools", "membench.cu")
LIB = os.path.join(ROOT, "tools", "libmembench.so")


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                               "-fPIC", "-cudart=static", "-o", LIB, SRC])
    return ctypes.CDLL(LIB)


def main():
    L = build()
    L.membench_rw.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_longlong] * 2 + [ctypes.c_void_p, ctypes.c_int,
                                                                                   ctypes.c_int, ctypes.c_int,
                                                                                   ctypes.c_void_p]
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    sink = torch.zeros(8, dtype=torch.int32, device="cuda")
    cases = [("C2", 18.9e6, 29.4e6), ("C3", 60.1e6, 22.0e6), ("C4", 184.5e6, 117.4e6), ("C5", 1028.8e6, 176.1e6),
             ("copy48", 24e6, 24e6), ("copy2G", 1e9, 1e9)]
    for name, rd, wr in cases:
        rd, wr = int(rd) // 32 * 32, int(wr) // 32 * 32
        n_sets = max(2, math.ceil(3 * l2 / (rd + wr)))
        bufs = [(torch.empty(rd, dtype=torch.uint8, device="cuda"), torch.empty(wr, dtype=torch.uint8, device="cuda"))
                for _ in range(n_sets)]
        for pdl in (0, 1):
            for blocks_per_sm in (4, 8):
                blocks, threads = 148 * blocks_per_sm, 256
                s = torch.cuda.Stream()

                def step(i):
                    b = bufs[i % n_sets]
                    e = L.membench_rw(b[0].data_ptr(), b[1].data_ptr(), rd, wr, sink.data_ptr(), blocks, threads,
                                      pdl, s.cuda_stream)
                    assert e == 0, e
                steps = 200 if rd + wr < 4e8 else 20
                with torch.cuda.stream(s):
                    for i in range(3):
                        step(i)
                s.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    with torch.cuda.graph(g, stream=s):
                        for i in range(steps):
                            step(i)
                s.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    g.replay()
                    e0.record(s)
                    for _ in range(5):
                        g.replay()
                    e1.record(s)
                s.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / (5 * steps)
                print(f"{name:7s} rd {rd / 1e6:7.1f} MB wr {wr / 1e6:7.1f} MB pdl={pdl} blocks={blocks:5d}: "
                      f"{us:8.2f} us  {(rd + wr) / us / 1e3:7.1f} GB/s", flush=True)
        del bufs




def bulk_main():
    L = build()
    L.membench_bulk.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_int, ctypes.c_void_p]
    sink = torch.zeros(8, dtype=torch.int32, device="cuda")
    nbytes = 1 << 30
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for chunk, per in [(16384, 1), (32768, 1), (49152, 1), (16384, 32), (32768, 64), (49152, 96), (49152, 384)]:
        for bps in (1, 2):
            blocks = 148 * bps
            with torch.cuda.stream(s):
                L.membench_bulk(src.data_ptr(), nbytes, chunk, per, sink.data_ptr(), blocks, s.cuda_stream)
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(3):
                    L.membench_bulk(src.data_ptr(), nbytes, chunk, per, sink.data_ptr(), blocks, s.cuda_stream)
                e1.record(s)
            s.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 3
            print(f"bulk read: chunk {chunk:6d} B in {per:3d} copies of {chunk // per:5d} B, {blocks} CTAs x 4 stages: "
                  f"{nbytes / us / 1e3:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    bulk_main() if "bulk" in sys.argv else main()
