"""Measure the int8 tensor-core rate on this B200 (torch._int_mm -> cuBLASLt, kind::i8)."""
import json, torch
a = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (8192, 8192), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
best = 1e9
for _ in range(10):
    s.record(); torch._int_mm(a, b); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
print(json.dumps({"int8_tops": 2 * 8192**3 / best / 1e9, "ms": best}))
