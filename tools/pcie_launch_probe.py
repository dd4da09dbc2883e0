"""Does PCIe copy traffic slow a chain of dependent kernel launches, and does a CUDA graph avoid it?
A chain of 200 dependent fp64 512x512 matmuls (~10 us each), eager vs replayed from a graph, timed
alone and while a copier thread streams 84 MB D2H (or 17 MB H2D) copies back to back."""
import json
import sys
import threading
import time

import torch

DIR = sys.argv[1] if len(sys.argv) > 1 else "d2h"
a = torch.randn(512, 512, dtype=torch.float64, device="cuda") / 40
x = torch.randn(512, 512, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()


def chain():
    y = x
    for _ in range(200):
        y = a @ y
    return y


with torch.cuda.stream(s):
    chain()
s.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    chain()


def t_eager():
    with torch.cuda.stream(s):
        chain()
    s.synchronize()


def t_graph():
    with torch.cuda.stream(s):
        g.replay()
    s.synchronize()


def rate(fn, reps=20):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


cst = torch.cuda.Stream()
h = torch.empty(84 * 2 ** 20 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(h, device="cuda")
stop = threading.Event()


def copier():
    while not stop.is_set():
        with torch.cuda.stream(cst):
            if DIR == "d2h":
                h.copy_(d, non_blocking=True)
            else:
                d.copy_(h, non_blocking=True)
        cst.synchronize()


res = {"dir": DIR, "eager_ms_alone": rate(t_eager), "graph_ms_alone": rate(t_graph)}
th = threading.Thread(target=copier)
th.start()
time.sleep(0.05)
res["eager_ms_with_copies"] = rate(t_eager)
res["graph_ms_with_copies"] = rate(t_graph)
stop.set()
th.join()
print(json.dumps(res))
