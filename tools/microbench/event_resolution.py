import torch
x = torch.empty(1, device="cuda")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2000)]
big = torch.empty(2**24, device="cuda")
for i, (a, b) in enumerate(ev):
    a.record(); big[: (i % 50 + 1) * 20000].add_(1.0); b.record()
torch.cuda.synchronize()
vals = sorted(set(round(a.elapsed_time(b) * 1e3, 3) for a, b in ev))
print("distinct elapsed values (us):", vals[:40])
