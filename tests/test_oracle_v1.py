"""CPU pin of the reference-readable (version 1) restatement: the oracle's
chunk-restart archives (fmt 3: the reference's exact SZ chain with a forced
escape every 16384 values) are deserialised and decoded by the unmodified
reference package to the oracle's values, within the bound.  The GPU writer
is byte-identical to this restatement (tests/test_gpu_v1.py)."""

import os
import sys

import numpy as np
import pytest

from paper_1711_03888_b200 import datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "nbz")):
            os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbz_numba_cache")
            if path not in sys.path:
                sys.path.insert(0, path)
            try:
                import nbz
                from nbz import io
                return nbz, io
            except Exception:  # pragma: no cover
                return None
    return None


@pytest.mark.parametrize("mode", ["sz-lv", "sz-lv-prx"])
@pytest.mark.parametrize("case", ["hacc", "amdf", "noise"])
def test_restart_chain_archive_reads_in_reference(oracle_lib, mode, case):
    r = _reference()
    if r is None:
        pytest.skip("reference package not available")
    ref_nbz, ref_io = r
    O = oracle_lib
    if case == "hacc":
        fields = datagen.small_hacc(36)            # 46656 values: 3 chunks, ragged
    elif case == "amdf":
        fields = datagen.small_amdf(40000)
    else:
        rng = np.random.default_rng(3)
        fields = [rng.standard_cauchy(20000).astype(np.float32) for _ in range(6)]
    out = O.compress(fields, mode, "rel", 1e-4, fmt=3)
    wire = out["wire"]
    ar = ref_io.deserialize_archive(wire)
    got = list(ref_nbz.decompress(ar).fields())
    odec = O.decompress(wire)
    order = out["order"]
    for fi in range(6):
        assert np.array_equal(got[fi].view(np.uint32), odec[fi].view(np.uint32)), fi
        x = fields[fi] if order is None else fields[fi][order]
        assert np.abs(x.astype(np.float64) - got[fi].astype(np.float64)).max() <= out["bounds"][fi]
    # the size cost of the restarts: well inside the 0.5% ratio tolerance on
    # snapshot-like data (escape-heavy Cauchy noise re-chains differently)
    if case != "noise":
        v1 = O.compress(fields, mode, "rel", 1e-4, fmt=1)
        assert abs(out["ratio"] / v1["ratio"] - 1) < 0.005
