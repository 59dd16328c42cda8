"""peek_columns stage entry vs the oracle on random maps of several shapes; first mismatch."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07809_b200 import stereotk as stk
import oracle
port = oracle.port()
dev = stk.Device(0, 64, 64)
rng = np.random.default_rng(0)
for (H, W, p) in [(240, 320, 0.3), (2304, 64, 0.3), (4320, 64, 0.3), (4320, 64, 0.02), (2304, 64, 0.02), (700, 32, 0.01), (300, 32, 0.005)]:
    m = np.where(rng.random((H, W)) < p, rng.integers(0, 257, (H, W)), -1).astype(np.int16)
    got = stk.peek_columns(m, 1, device=dev)
    want = port.peek_columns(m, 1)
    bad = np.argwhere(got != want)
    print(H, W, p, "mismatches", len(bad))
    if len(bad):
        y, x = bad[0]
        col = m[:, x]
        print(" first", y, x, "got", got[y, x], "want", want[y, x], "known rows", np.nonzero(col >= 0)[0][:10], col[col >= 0][:10])
