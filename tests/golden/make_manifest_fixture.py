"""Build the manifest fixture of the CSR-system tests from the reference itself
(run in the build container, where /root/reference exists; the GPU box only
reads the committed output).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_manifest_fixture.py

Writes tests/golden/manifest_c6/ (the reference's export_model of
builtin_model(cells=6): five Matrix Market blocks and manifest.json) and
tests/golden/manifest_c6_ref.npz (the blocks as the reference's load_model
returns them, CsrMatrix arrays, plus exponential_ramp at a few times).
"""
import shutil
from pathlib import Path

import numpy as np
from mqsolve import builtin_model
from mqsolve.bench import load_model
from mqsolve.model import export_model

here = Path(__file__).resolve().parent
out = here / "manifest_c6"
if out.exists():
    shutil.rmtree(out)
model = builtin_model(cells=6)
export_model(model, out)
# drop the builtin section: the stored blocks define a frozen-linear system
import json  # noqa: E402
mf = json.loads((out / "manifest.json").read_text())
mf.pop("builtin", None)
(out / "manifest.json").write_text(json.dumps(mf, indent=1, sort_keys=True) + "\n")
system, m, _ = load_model(out)
assert m is None
arrays = {}
for name, blk in (("m_c", system.mc), ("k_cn", system.kcn), ("k_n", system.kn)):
    arrays[f"{name}_rp"] = np.asarray(blk.row_ptr)
    arrays[f"{name}_ci"] = np.asarray(blk.col_idx)
    arrays[f"{name}_va"] = np.asarray(blk.values)
kc = system.kc_matrix(np.zeros(system.n_c))
arrays["k_c_rp"], arrays["k_c_ci"], arrays["k_c_va"] = (np.asarray(kc.row_ptr), np.asarray(kc.col_idx),
                                                       np.asarray(kc.values))
arrays["pattern"] = np.asarray(system.source.pattern)
ts = np.array([0.0, 1e-4, 3.3e-3, 0.02])
arrays["ramp_t"] = ts
arrays["ramp_w"] = np.array([system.source.waveform(t) for t in ts])
np.savez_compressed(here / "manifest_c6_ref.npz", **arrays)
print(out, {k: v.shape for k, v in arrays.items()})
