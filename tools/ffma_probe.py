"""Run the FP32 FFMA-peak probe kernel (the roofline denominator, spc_ffma_peak_kernel)
a few times; under ncu its FMA-pipe utilisation shows whether it saturates the pipe."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_10175_b200 as sp  # noqa: E402

L = sp._lib.load()
buf = torch.zeros(16, device="cuda")
fl = ctypes.c_double()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(3):
    e0.record(st)
    L.spc_ffma_peak_kernel(ctypes.c_void_p(buf.data_ptr()), 148 * 16, 4096, ctypes.byref(fl), ctypes.c_void_p(st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    print(f"ffma probe: {fl.value / (e0.elapsed_time(e1) * 1e-3) / 1e12:.2f} TFLOP/s")
