"""D2H copy bandwidth of the e2e step's two outputs (420 MB positions + 558 MB faces) to pinned host
memory: sequential vs two streams vs chunked (is the e2e step at the PCIe ceiling?)."""
import torch, time
a = torch.empty(420_000_000 // 4, dtype=torch.float32, device="cuda").fill_(1)
b = torch.empty(558_000_000 // 4, dtype=torch.int32, device="cuda").fill_(2)
ha = torch.empty_like(a, device="cpu").pin_memory(); hb = torch.empty_like(b, device="cpu").pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    ha.copy_(a, non_blocking=True); hb.copy_(b, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): ha.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): hb.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter() - t
    # chunked on two streams
    t = time.perf_counter()
    n = a.numel() // 2; m = b.numel() // 2
    with torch.cuda.stream(s1): ha[:n].copy_(a[:n], non_blocking=True); hb[:m].copy_(b[:m], non_blocking=True)
    with torch.cuda.stream(s2): ha[n:].copy_(a[n:], non_blocking=True); hb[m:].copy_(b[m:], non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter() - t
    print(f"seq {t1*1e3:.2f} ms ({0.978/t1:.1f} GB/s)  2 streams {t2*1e3:.2f} ms ({0.978/t2:.1f} GB/s)  chunked {t3*1e3:.2f} ms")
