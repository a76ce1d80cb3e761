"""Host-side trace rendering against the reference (no GPU).

schur.trace_bytes must render a TransientResult exactly as the reference's
bench.trace_bytes (bench.py:341-357): rebuilt from the reference's own
columns (tests/golden/reference_trace.npz), the CSV is byte-identical.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_1611_06721_b200.schur import TRACE_HEADER, TransientResult, trace_bytes

GOLD = Path(__file__).parent / "golden" / "reference_trace.npz"
RUNS = ["cspe_100_1", "pod_30_1", "previous_30_1", "cspe_30_3", "pod_30_3"]


@pytest.mark.parametrize("key", RUNS)
def test_trace_bytes_identical_to_reference(key):
    g = np.load(GOLD)
    res = TransientResult(times=g[f"{key}_times"], probe_b=g[f"{key}_probe_b"], iters_src=g[f"{key}_iters_src"],
                          iters_cpl_prev=g[f"{key}_iters_cpl_prev"], iters_cpl_cur=g[f"{key}_iters_cpl_cur"],
                          basis_cols=g[f"{key}_basis_cols"], pod_k=g[f"{key}_pod_k"],
                          pod_info=g[f"{key}_pod_info"], final_a_c=g[f"{key}_final_a_c"],
                          final_a_n=g[f"{key}_final_a_n"])
    assert trace_bytes(res) == bytes(g[f"{key}_trace"])
    assert trace_bytes(res).decode().splitlines()[0] == TRACE_HEADER


def test_reference_trace_window_semantics():
    """What the device log must reproduce (schur.py:448-467, 524-538): the
    CSPE basis grows one column per step up to max_cols; POD rows with a
    three-step window report the window maximum of pod_k."""
    g = np.load(GOLD)
    assert list(g["cspe_100_1_basis_cols"][:7]) == [0, 1, 2, 3, 4, 5, 5]
    assert g["pod_30_3_pod_k"].max() > g["pod_30_3_basis_cols"].max() or \
        np.any(g["pod_30_3_pod_k"] > g["pod_30_3_basis_cols"])


def test_empty_trace_refused():
    z = np.zeros(0)
    with pytest.raises(ValueError):
        trace_bytes(TransientResult(z, z, z, z, z, z, z, z, z, None))
