"""Python-side cost of one bench step outside the native call (debug tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import timeline as T  # noqa: E402
import torch  # noqa: E402
from paper_2603_07156_b200 import session as S  # noqa: E402

orig = S.Ops.inner_iteration
acc = [0.0]
def wrapped(self, *a, **k):
    t0 = time.perf_counter()
    r = orig(self, *a, **k)
    acc[0] += time.perf_counter() - t0
    return r
S.Ops.inner_iteration = wrapped
for _ in range(5):
    T.step()
torch.cuda.synchronize()
acc[0] = 0.0
N = 200
t0 = time.perf_counter()
for _ in range(N):
    T.step()
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / N * 1e6
print(f"step wall {tot:.1f} us; inside otb_inner_iteration {acc[0] / N * 1e6:.1f} us; Python outside {tot - acc[0] / N * 1e6:.1f} us")
