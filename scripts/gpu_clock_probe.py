"""Clock / power under sustained load for our GEMM vs cuBLAS (is the pair
kernel at the 1 kW power cap?)."""
import os, sys, threading, time, statistics
sys.path.insert(0, ".")
import torch, pynvml
import paper_2003_06324_b200 as fi

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)

def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.01)

def run(name, fn, flops, secs=1.5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    out, stop = [], threading.Event()
    t = threading.Thread(target=sample, args=(stop, out)); t.start()
    n = 0; t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < secs:
        for _ in range(20): fn()
        n += 20
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); t.join()
    ms = e0.elapsed_time(e1) / n
    clk = statistics.median([o[0] for o in out[5:]]); pw = statistics.median([o[1] for o in out[5:]])
    reasons = 0
    for o in out[5:]: reasons |= o[2]
    print(f"{name:40s} {flops/ms/1e9:7.1f} TF  clk {clk:6.0f} MHz  power {pw:6.0f} W  reasons 0x{reasons:x}  "
          f"TF/GHz {flops/ms/1e9/clk*1000:6.1f}", flush=True)

for (m, n, k) in [(4096, 4096, 4096), (8192, 8192, 8192)]:
    for pair, tn in [(True, 256), (False, 256)]:
        for sk in ["0", "1"]:
            os.environ["FI_STREAMK"] = sk
            plan = fi.Plan(fi.strategies.tc_strategy(m, n, k, pair=pair, tile_n=tn))
            A = torch.randn(k, m, device="cuda").half(); B = torch.randn(n, k, device="cuda").half()
            C = torch.empty(n, m, device="cuda")
            s = torch.cuda.current_stream().cuda_stream
            run(f"ours {m} pair={pair} tn={tn} sk={plan.info.streamk}",
                lambda: plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s), plan.flops)
    a = torch.randn(m, k, device="cuda").half(); b = torch.randn(k, n, device="cuda").half()
    run(f"cuBLAS {m}", lambda: torch.matmul(a, b), 2.0 * m * n * k)
