"""cProfile of the host side of bench steps (cfg2): where the Python time
between kernel launches goes (debug tool)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import timeline as T  # noqa: E402  (builds the cfg2 state; its own profile runs on import)

import torch  # noqa: E402

for _ in range(3):
    T.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    T.step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
