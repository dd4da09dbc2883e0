"""PCIe-only ceiling of the e2e leg: the transfers of one config-2 phi_0..phi_4 call (b in: 17.2 MB;
phi_0..phi_4 out: 83.9 MB, pinned host buffers) repeated by K host threads on their own streams with
no compute. actions/s here bounds the e2e value from above whatever the kernels do."""
import json
import sys
import threading
import time

import torch

N = 128 ** 3
K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
REPS = 20
callers = []
for _ in range(K):
    st = torch.cuda.Stream()
    hb = torch.empty(N + 1024, dtype=torch.float64).pin_memory()  # b + factors
    ho = torch.empty(5 * N, dtype=torch.float64).pin_memory()
    db = torch.empty_like(hb, device="cuda")
    do = torch.empty_like(ho, device="cuda")
    callers.append((st, hb, ho, db, do))


def one(c):
    st, hb, ho, db, do = c
    with torch.cuda.stream(st):
        db.copy_(hb, non_blocking=True)
        ho.copy_(do, non_blocking=True)
    st.synchronize()


def worker(c):
    for _ in range(REPS):
        one(c)


for c in callers:
    one(c)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(REPS):
    one(callers[0])
t1 = time.perf_counter() - t0
t0 = time.perf_counter()
ths = [threading.Thread(target=worker, args=(c,)) for c in callers]
[t.start() for t in ths]
[t.join() for t in ths]
tk = time.perf_counter() - t0
mb = (N + 1024 + 5 * N) * 8 / 1e6
print(json.dumps({"MB_per_action": mb, "single_actions_per_s": REPS / t1, "callers": K,
                  "concurrent_actions_per_s": K * REPS / tk, "concurrent_GBps": K * REPS * mb / tk / 1e3}))
