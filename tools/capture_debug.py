"""Debug: where the zero1 graph capture gets invalidated (after test_gpu_config1 + the allreduce case).
Driver-level stream capture status after each of our launches."""
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import driver as drv  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402

orig_check = _lib.check
log = []


def cap():
    err, st = drv.cuStreamIsCapturing(torch.cuda.current_stream().cuda_stream)
    return int(err), int(st)


def check(st, what):
    e, c = cap()
    if c != 0:
        log.append((what, st, e, c))
        if (c == 2 or st) and not getattr(check, "done", False):
            check.done = True
            print("FIRST BAD:", what, "status", st, "cap", (e, c), "prev:", log[-6:-1], flush=True)
            traceback.print_stack(limit=10)
    return orig_check(st, what)


_lib.check = check
import pytest  # noqa: E402
rc = pytest.main(["-q", "-p", "no:cacheprovider", "-x", "-s", "tests/test_gpu_config1.py", "tests/test_gpu_graph_dp.py"])
print("rc", rc)
