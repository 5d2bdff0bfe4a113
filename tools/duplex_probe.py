"""PCIe duplex probe: H2D and D2H copies alone, back to back, and concurrently on two streams."""
import time, torch
dev = torch.device("cuda", 0)
n_up, n_dn = 2 << 30, 1 << 30
hu = torch.empty(n_up, dtype=torch.uint8).pin_memory(); du = torch.empty(n_up, dtype=torch.uint8, device=dev)
hd = torch.empty(n_dn, dtype=torch.uint8).pin_memory(); dd = torch.empty(n_dn, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(up, dn, conc):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if up:
        with torch.cuda.stream(s1): du.copy_(hu, non_blocking=True)
    if not conc: torch.cuda.synchronize()
    if dn:
        with torch.cuda.stream(s2): hd.copy_(dd, non_blocking=True)
    torch.cuda.synchronize(); return 1e3 * (time.perf_counter() - t0)
for it in range(3):
    print("up 2GB %.1f ms | down 1GB %.1f ms | sequential %.1f ms | concurrent %.1f ms" % (run(1, 0, 0), run(0, 1, 0), run(1, 1, 0), run(1, 1, 1)), flush=True)
