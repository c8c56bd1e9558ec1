"""PCIe copy-engine probe: H2D alone, D2H alone, both concurrently (pinned),
whole 64 MiB copies and 8 MiB chunks."""
import torch, time
n = 64 << 20  # 64 MiB
h_up = torch.empty(n // 4, dtype=torch.float32, pin_memory=True).fill_(1)
h_dn = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d_up = torch.empty(n // 4, device="cuda"); d_dn = torch.ones(n // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(up, dn, chunks=1, reps=10):
    c = n // 4 // chunks
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        for i in range(chunks):
            if up:
                with torch.cuda.stream(s1): d_up[i*c:(i+1)*c].copy_(h_up[i*c:(i+1)*c], non_blocking=True)
            if dn:
                with torch.cuda.stream(s2): h_dn[i*c:(i+1)*c].copy_(d_dn[i*c:(i+1)*c], non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps
for ch in (1, 8):
    for _ in range(2): run(1, 1, ch)
    tu, td, tb = run(1, 0, ch), run(0, 1, ch), run(1, 1, ch)
    print(f"chunks={ch}: H2D {n/tu/1e9:.1f} GB/s  D2H {n/td/1e9:.1f} GB/s  both: {2*n/tb/1e9:.1f} GB/s total ({tb*1e3:.2f} ms for 2x64 MiB)")
# timed with events per direction
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
torch.cuda.synchronize()
s1.record_event(e[0]); s2.record_event(e[2])
with torch.cuda.stream(s1): d_up.copy_(h_up, non_blocking=True)
with torch.cuda.stream(s2): h_dn.copy_(d_dn, non_blocking=True)
s1.record_event(e[1]); s2.record_event(e[3])
torch.cuda.synchronize()
print(f"events: H2D {e[0].elapsed_time(e[1]):.3f} ms, D2H {e[2].elapsed_time(e[3]):.3f} ms, D2H start after H2D start {e[0].elapsed_time(e[2]):.3f} ms")
