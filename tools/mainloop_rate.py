"""Main-loop rate of the leaf kernel (mk_dgemm, 4 whole waves, K = 8192 and 16384) with the SM
clock sampled via NVML during the run. Dev tool for A/B of kernel env knobs."""
import os, sys, threading, time
import torch
sys.path.insert(0, "tools")
import quick_gpu as q
import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk, stop = [], False


def sample():
    while not stop:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.01)


SM = torch.cuda.get_device_properties(0).multi_processor_count
M, N = SM * 128, int(os.environ.get("WAVES", "4")) * 128
res = {}
th = threading.Thread(target=sample); th.start()
for K in (8192, 16384):
    a = torch.randn(M, K, device="cuda", dtype=torch.float64)
    b = torch.randn(K, N, device="cuda", dtype=torch.float64)
    c = torch.empty(M, N, device="cuda", dtype=torch.float64)
    res[K] = q.timeit(lambda: q.dgemm(a, b, c), reps=40, warm=5)
stop = True; th.join()
sl = (res[16384] - res[8192]) / 8192
clk.sort()
q.out(tag=os.environ.get("TAG", ""), ms8k=round(res[8192], 4), ms16k=round(res[16384], 4),
      mainloop_tflops=round(2 * M * N / sl / 1e9, 3), intercept_us=round((res[8192] - 8192 * sl) * 1e3, 2),
      sm_mhz_median=clk[len(clk) // 2] if clk else None, sm_mhz_min=clk[0] if clk else None)
