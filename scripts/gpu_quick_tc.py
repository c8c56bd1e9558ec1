"""Quick GPU check of the raw tcgen05 GEMM family against torch (fp32 ref)."""
import ctypes as C
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2003_06324_b200 import _native as N

def run(cfg, M, Nn, K, dtype=torch.float16, a_row=0, b_row=0, c_row=0, c_elem=0, reps=0):
    torch.manual_seed(0)
    A = torch.randint(-3, 4, (M, K), device="cuda").to(dtype)
    B = torch.randint(-3, 4, (K, Nn), device="cuda").to(dtype)
    # physical layouts: row-major tensors for row layouts, transposed-contiguous for col-major
    Ad = A.contiguous() if a_row else A.t().contiguous()
    Bd = B.contiguous() if b_row else B.t().contiguous()
    cdt = {0: torch.float32, 1: torch.float16, 2: torch.bfloat16}[c_elem]
    Cd = torch.full((M, Nn) if c_row else (Nn, M), float("nan"), device="cuda", dtype=cdt)
    lda = K if a_row else M
    ldb = Nn if b_row else K
    ldc = Nn if c_row else M
    c = N.TcConfig(cfg[0], cfg[1], cfg[2], N.FI_BF16 if dtype == torch.bfloat16 else N.FI_F16,
                   a_row, b_row, c_row, c_elem, 8, 0)
    st = torch.cuda.current_stream().cuda_stream
    r = N.lib.fi_tc_gemm(C.byref(c), Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr(), M, Nn, K,
                         lda, ldb, ldc, None, st)
    if r != 0:
        return f"status {r}: {N.last_error()}"
    torch.cuda.synchronize()
    got = Cd if c_row else Cd.t()
    ref = A.float() @ B.float()
    err = (got.float() - ref).abs().max().item()
    out = f"maxerr {err:.3g}"
    if reps:
        for _ in range(3):
            N.lib.fi_tc_gemm(C.byref(c), Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr(), M, Nn, K, lda, ldb, ldc, None, st)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            N.lib.fi_tc_gemm(C.byref(c), Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr(), M, Nn, K, lda, ldb, ldc, None, st)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out += f"  {ms*1e3:.1f} us  {2*M*Nn*K/ms/1e9:.1f} TFLOP/s"
    return out

if __name__ == "__main__":
    print(N.lib.fi_version().decode(), torch.cuda.get_device_name())
    cases = []
    for cfg in [(1, 128, 1), (1, 256, 1), (1, 64, 1), (2, 256, 1), (2, 128, 1)]:
        for (ar, br) in [(0, 0), (1, 0), (0, 1), (1, 1)]:
            cases.append((cfg, 512, 512, 256, ar, br))
    for cfg, M, Nn, K, ar, br in cases:
        print(cfg, M, Nn, K, "a_row", ar, "b_row", br, "->", run(cfg, M, Nn, K, a_row=ar, b_row=br), flush=True)
    for cfg in [(1, 128, 2), (1, 128, 4), (1, 64, 2), (1, 256, 2), (1, 256, 4), (2, 256, 2), (2, 256, 4), (2, 128, 2), (2, 128, 4)]:
        print(cfg, "splitk 512x512x1024 ->", run(cfg, 512, 512, 1024), flush=True)
    print("c_row f16 out:", run((2, 256, 1), 512, 512, 256, c_row=1, c_elem=1))
    print("bf16 in:", run((2, 256, 1), 512, 512, 256, dtype=torch.bfloat16))
    for cfg in [(1, 256, 1), (2, 256, 1), (2, 128, 1)]:
        print("perf 8192", cfg, run(cfg, 8192, 8192, 8192, reps=10), flush=True)
        print("perf 4096", cfg, run(cfg, 4096, 4096, 4096, reps=20), flush=True)
    for cfg in [(1, 128, 2), (1, 128, 4), (1, 256, 4), (2, 256, 2), (2, 256, 4), (2, 128, 2), (2, 128, 4)]:
        print("perf splitk 1024x1024x32768", cfg, run(cfg, 1024, 1024, 32768, reps=20), flush=True)
    # torch reference speed
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.float16); b = torch.randn(8192, 8192, device="cuda", dtype=torch.float16)
    for _ in range(3): a @ b
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"torch/cuBLAS 8192^3 f16: {2*8192**3/ms/1e9:.1f} TFLOP/s")
