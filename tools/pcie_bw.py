import torch, time
n = 233570304 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
o = torch.empty(103809024 // 2, dtype=torch.bfloat16, device="cuda")
ho = torch.empty(103809024 // 2, dtype=torch.bfloat16).pin_memory()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D 234 MB: {ms:.3f} ms = {233570304/ms/1e6:.1f} GB/s")
e0.record()
for _ in range(10):
    ho.copy_(o, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"D2H 104 MB: {ms:.3f} ms = {103809024/ms/1e6:.1f} GB/s")
# both directions at once (the host-buffer pipeline's steady state)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(o, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D 234 MB + D2H 104 MB concurrently: {ms:.3f} ms per pair")
