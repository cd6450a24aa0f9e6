"""As e2e_cold3.py, with the CUDA context already created by torch (bench.py's situation)."""
import os
import sys
import time
import torch
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = [sys.argv[0]]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "e2e_cold3.py")).read())
