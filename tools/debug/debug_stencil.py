import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2109_05410_b200 import oocz as Z
n, planes = 64, 40
u = torch.rand(planes, n, n, device="cuda"); up = u.clone(); m = torch.full_like(u, 0.1)
try:
    Z.oocz_stencil_step_planes(u, up, m, n, n, planes, Z.default_coeffs(), 4, planes - 4, 0, planes, None)
    torch.cuda.synchronize(); print("ok")
except Exception as e:
    print("ERR", e)
