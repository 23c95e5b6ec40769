"""cuBLAS bf16 8192^3 reference launch for ncu comparisons with sim_tc_kernel."""
import torch
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(20):
    c = a @ b
torch.cuda.synchronize()
