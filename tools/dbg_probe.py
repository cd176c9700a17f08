import sys, os
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "oracle")]
import numpy as np, oracle
from paper_2210_15962_b200 import _kernels, _lib
_lib.set_variant(_lib.VARIANT_FAST)
for L in (3, 5, 27, 101, 201):
    d = (L + 1) // 2
    rng = np.random.default_rng(1)
    halves = np.stack([np.ones(d), rng.choice([-1, 1], size=d)]).astype(np.int8)
    got = _kernels.eval_states(L, halves)
    for i in range(2):
        s, c, _ = oracle.init_state(L, halves[i].astype(np.int64))
        want = oracle.all_neighbor_deltas(L, s, c)
        print(L, i, "OK" if np.array_equal(got[i, 0], want) else "BAD", got[i, 0][:8].tolist(), want[:8].tolist(), flush=True)
