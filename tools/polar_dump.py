"""Dump device polar rotations for the test cases (debugging aid): gpurun_out/polar_<dtype>.npz"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_polar import _cases
from paper_2306_09021_b200.pbng import test_polar
F = _cases()
for dt in ("f64", "f32"):
    R = test_polar(F, dt)
    np.savez_compressed(f"gpurun_out/polar_{dt}.npz", F=F, R=R)
print("ok")
