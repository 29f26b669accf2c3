"""The package's synthetic trace generator (synth.py) against the
reference's own bytes: the KSCD conformance fixture (with X/Y hidden states)
and the generator hashes frozen in golden.json.  CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2512_16391_b200 import kscd_io
from paper_2512_16391_b200.exceptions import InvalidArgumentError
from paper_2512_16391_b200.synth import SynthConfig, generate_synthetic


def test_conformance_fixture_bytes(tmp_path):
    t = generate_synthetic(SynthConfig(2, 2, 1, 4, 3, seed=42, layer_correlation=0.5, include_xy=True,
                                       prompt_id="conformance-v1"))
    p = tmp_path / "c.kscd"
    kscd_io.write_trace(p, t)
    with open(os.path.join(GOLDEN, "conformance_v1.kscd"), "rb") as f:
        want = f.read()
    assert p.read_bytes() == want


def test_generator_hashes_match_reference():
    meta = json.load(open(os.path.join(GOLDEN, "golden.json")))
    for name, ent in meta["synth_sha256"].items():
        a = ent["args"]
        t = generate_synthetic(SynthConfig(a["L"], a["Hq"], a["Hkv"], a["d"], a["N"], seed=a["seed"],
                                           layer_correlation=a["rho"], head_permutations=a.get("perms")))
        h = hashlib.sha256()
        for arr in (t.Q, t.K, t.V):
            h.update(np.ascontiguousarray(arr).tobytes())
        assert h.hexdigest() == ent["sha256"], name


def test_validation():
    with pytest.raises(InvalidArgumentError):
        generate_synthetic(SynthConfig(2, 3, 2, 4, 3))
    with pytest.raises(InvalidArgumentError):
        generate_synthetic(SynthConfig(2, 2, 1, 4, 3, layer_correlation=1.5))
    with pytest.raises(InvalidArgumentError):
        generate_synthetic(SynthConfig(2, 2, 2, 4, 3, head_permutations=[[0, 1], [0, 0]]))
