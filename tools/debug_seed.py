"""Dev tool: locate the first K-means++ slot where GPU and CPU checkers diverge."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1])); sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import paper_2311_04517_b200 as hp
from oracle_py import orc, ref
from test_parity_gpu import mixture

dtype, n, k, s, npend = np.float32, 16, 10, 20000, 10
X = mixture(s, n, k, seed=21 + k, dtype=dtype)
Xw = X.astype(np.float64)
init = np.zeros((k, n)); deg = np.ones(k, np.uint8)
for kk in range(1, k + 1):
    g = hp.kmeanspp_seed(X, kk, hp.SeedConfig(), hp.RngStream(1234 + k))[0]
    o = orc().reinit(Xw, np.zeros((kk, n)), np.ones(kk, np.uint8), orc().rng(seed=1234 + k))[0]
    R = ref()
    r = R.reinit(Xw, np.zeros((kk, n)), np.ones(kk, np.uint8), R.rng(seed=1234 + k))[0] if R else o
    gi = [int(np.where((Xw == c).all(1))[0][0]) for c in g]
    oi = [int(np.where((Xw == c).all(1))[0][0]) for c in o]
    ri = [int(np.where((Xw == c).all(1))[0][0]) for c in r]
    print(kk, "gpu", gi, "orc", oi, "ref", ri, "OK" if gi == oi == ri else "DIFF")
    if gi != oi:
        # replay the oracle's slot with the reference draws and print candidate costs
        rng = hp.RngStream(1234 + k)
        first = rng.uniform_index(s)
        units = rng.units(3 * (kk - 1))
        d2 = np.full(s, np.inf)
        chosen = [first]
        d2 = np.minimum(d2, ((Xw - Xw[first]) ** 2).sum(1))
        for t in range(kk - 1):
            cum = np.cumsum(d2)
            cands = [int(np.searchsorted(cum, u * cum[-1], side="right")) for u in units[3 * t: 3 * t + 3]]
            costs = [np.minimum(d2, ((Xw - Xw[c]) ** 2).sum(1)).sum() for c in cands]
            b = int(np.argmin(costs))
            print("  slot", t + 1, "cands", cands, "costs", costs, "u*tot", [u * cum[-1] for u in units[3*t:3*t+3]])
            d2 = np.minimum(d2, ((Xw - Xw[cands[b]]) ** 2).sum(1))
        break
