"""The 125M 'converge' run (configs[2]) on the GPU vs the committed CPU reference
curve: smoothed curves and the relative gap every 10 steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import test_gpu_llama as T  # noqa: E402

gpu, ref, gpu_s, ref_s, gap, run = T._run_125m(sys.argv[1] if len(sys.argv) > 1 else "converge")
for i in range(0, run["steps"], 10):
    print(f"step {i:3d}  gpu {gpu[i]:.4f} ref {ref[i]:.4f}  smoothed gpu {gpu_s[i]:.4f} ref {ref_s[i]:.4f}  gap {gap[i]:.4f}")
print(f"final smoothed gap {gap[-1]:.4f}; max after step 40: {gap[40:].max():.4f} at {40 + int(gap[40:].argmax())}; "
      f"max after step 100: {gap[100:].max():.4f}")
