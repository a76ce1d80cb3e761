"""Sharded step at 1 and N ranks: the CSPE caches after one step (diagnostic).

    python tools/sharded_cache_check.py --config 4 --world 2
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--world", type=int, default=2)
    args = ap.parse_args()
    import numpy as np

    from paper_1611_06721_b200 import configs as C
    from paper_1611_06721_b200.slabstep import SlabStepper
    spec = C.config_spec(args.config)
    prob = C.make_problem(args.config)
    res = {}
    caches = {}
    for w in (1, args.world):
        st = SlabStepper(prob, w, strategy="cspe", max_cols=5)
        r1, r2 = st.step(spec.dt)
        fams = {}
        for fam in (0, 1, 2):
            parts = [s.cspe_export(fam) for s in st.slabs]
            k = parts[0][0].shape[1]
            U = np.zeros((st.n_n, k))
            KU = np.zeros((st.n_n, k))
            for s, (u, ku, g) in zip(st.slabs, parts):
                U[s.gidx] = u
                KU[s.gidx] = ku
            fams[fam] = (U, KU, [p[2] for p in parts])
        caches[w] = fams
        res[f"w{w}_iters"] = [r1.iterations, r2.iterations]
        st.close()
    for fam in (0, 1, 2):
        U1, KU1, G1 = caches[1][fam]
        U2, KU2, G2 = caches[args.world][fam]
        d = {"k": [U1.shape[1], U2.shape[1]], "G1": [g.tolist() for g in G1], "G2": [g.tolist() for g in G2]}
        if U1.shape == U2.shape and U1.size:
            d["U_rel"] = float(np.linalg.norm(U1 - U2) / np.linalg.norm(U1))
            d["KU_rel"] = float(np.linalg.norm(KU1 - KU2) / np.linalg.norm(KU1))
            q = int(np.argmax(np.abs(KU1 - KU2).max(axis=1)))
            d["worst_row"] = q
        res[f"fam{fam}"] = d
    print(json.dumps(res))


if __name__ == "__main__":
    main()
