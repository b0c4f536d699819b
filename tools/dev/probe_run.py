"""Run the UMMA/TMA/TMEM probe on cuda:0 and compare with torch (fp32)."""
import ctypes
import os
import sys

import torch

here = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(here, "_probe.so"))
lib.probe_run.restype = ctypes.c_int
lib.probe_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                          ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p]

torch.manual_seed(0)
dev = "cuda:0"
hq, qh = 2, 1
q = torch.randn(128, hq, 128, device=dev).to(torch.bfloat16)
k = torch.randn(128, 1, 128, device=dev).to(torch.bfloat16)
v = torch.randn(128, 1, 128, device=dev).to(torch.bfloat16)
s_out = torch.zeros(128, 128, device=dev)
o_out = torch.zeros(128, 128, device=dev)
pscale = 0.05
rc = lib.probe_run(q.data_ptr(), hq, qh, k.data_ptr(), v.data_ptr(), pscale, s_out.data_ptr(),
                   o_out.data_ptr())
torch.cuda.synchronize()
print("rc", rc)
s_ref = q[:, qh].float() @ k[:, 0].float().T
p = (s_ref * pscale).to(torch.bfloat16).float()
o_ref = p @ v[:, 0].float()
ds = (s_out - s_ref).abs().max().item()
do = (o_out - o_ref).abs().max().item()
print("S maxdiff", ds, "S scale", s_ref.abs().max().item())
print("O maxdiff", do, "O scale", o_ref.abs().max().item())
if ds > 1e-2:
    # diagnose: find permutation
    print("S[0,:8]", s_out[0, :8].tolist())
    print("ref[0,:8]", s_ref[0, :8].tolist())
    print("S[1,:8]", s_out[1, :8].tolist())
    print("ref[1,:8]", s_ref[1, :8].tolist())
if do > 1e-1:
    print("O[0,:8]", o_out[0, :8].tolist())
    print("ref[0,:8]", o_ref[0, :8].tolist())
ok = ds < 1e-2 and do < 5e-2
print("PROBE", "OK" if ok else "FAIL")
sys.exit(0 if ok else 1)
