"""PCIe: pitched (2D) H2D/D2H copies of 64 MiB with 2..64 KiB lines vs linear,
alone and with a concurrent linear copy in the other direction (pinned)."""
import ctypes, time
import torch
n = 64 << 20
h_a = torch.empty(n // 4, dtype=torch.float32, pin_memory=True).fill_(1)
h_c = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n // 4, device="cuda"); d_c = torch.ones(n // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
import glob
lib = ctypes.CDLL((glob.glob("/usr/local/cuda/lib64/libcudart.so.12*") or ["libcudart.so"])[0])
lib.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                  ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
def copy2d(dst, src, width_b, height, pitch_b, kind, stream):
    # cudaMemcpy2DAsync via the torch-bundled runtime
    return lib.cudaMemcpy2DAsync(dst, pitch_b, src, pitch_b, width_b, height, kind, stream)
ups = [torch.cuda.Stream() for _ in range(4)]
def run(seg, up=True, dn=False, reps=5, nstreams=1):
    pitch = 16384 * 4  # 64 KiB pitch (a 16384-row col-major matrix)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if up:
            if seg:  # 64 MiB in lines of `seg` bytes: several row panels side by side
                per = pitch // seg
                for p in range(per):
                    copy2d(d_a.data_ptr() + p * seg, h_a.data_ptr() + p * seg, seg, n // pitch, pitch, 1,
                           (ups[p % nstreams] if nstreams > 1 else s1).cuda_stream)
            else:
                with torch.cuda.stream(s1): d_a.copy_(h_a, non_blocking=True)
        if dn:
            with torch.cuda.stream(s2): h_c.copy_(d_c, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
for seg in (0, 2048, 4096, 8192, 16384, 65536):
    for _ in range(2): run(seg)
    tu = run(seg); tb = run(seg, dn=True)
    print(f"H2D lines {seg or 'linear':>6}: alone {n / tu / 1e9:5.1f} GB/s; with concurrent 64 MiB D2H: "
          f"{2 * n / tb / 1e9:5.1f} GB/s total ({tb * 1e3:.2f} ms)", flush=True)
for ns in (2, 4):
    for seg in (2048, 4096, 8192):
        for _ in range(2): run(seg, nstreams=ns)
        tu = run(seg, nstreams=ns); tb = run(seg, dn=True, nstreams=ns)
        print(f"{ns} streams, H2D lines {seg:>6}: alone {n / tu / 1e9:5.1f} GB/s; with concurrent 64 MiB D2H: "
              f"{2 * n / tb / 1e9:5.1f} GB/s total ({tb * 1e3:.2f} ms)", flush=True)
# D2H pitched lines with a concurrent linear H2D
def run_dn(seg, reps=5):
    pitch = 16384 * 4
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1): d_a.copy_(h_a, non_blocking=True)
        for p in range(pitch // seg):
            copy2d(h_c.data_ptr() + p * seg, d_c.data_ptr() + p * seg, seg, n // pitch, pitch, 2, s2.cuda_stream)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
for seg in (2048, 8192, 65536):
    for _ in range(2): run_dn(seg)
    tb = run_dn(seg)
    print(f"D2H lines {seg:>6} with concurrent linear H2D: {2 * n / tb / 1e9:5.1f} GB/s total", flush=True)
