"""Native listing front-end against the reference's
parse_kernels + soa.encode_cfg on the same listing texts (tests/golden/
make_front.py): identical SoA arrays, line tables, CFG diagnostics,
mnemonics and source locations, and identical ListingError messages on the
malformed listings."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

FIELDS = ("opclass", "block_of", "opnd_ptr", "opnd", "sync_kind", "sync_a", "sync_b", "blk_first",
          "blk_last", "succ_ptr", "succ", "pred_ptr", "pred", "unit_base", "offset", "line_id")


@pytest.fixture(scope="module")
def front_cases():
    z = np.load(GOLDEN / "front.npz")
    return json.loads(str(z["cases"])), json.loads(str(z["tables"]))


def test_native_front_matches_reference(front_cases):
    from paper_2604_20032_b200 import front
    cases, tables = front_cases
    assert len(cases) >= 150
    n_err = 0
    for c in cases:
        d = c["dialect"]
        if "error" in c:
            with pytest.raises(front.ListingError) as e:
                front.parse_kernels_soa(d, c["text"], tables[d])
            assert str(e.value) == c["error"], (c["text"], str(e.value), c["error"])
            n_err += 1
            continue
        got = front.parse_kernels_soa(d, c["text"], tables[d])
        assert list(got) == [k["name"] for k in c["kernels"]]
        for k in c["kernels"]:
            ks, meta = got[k["name"]]
            for f in FIELDS:
                assert np.array_equal(np.asarray(getattr(ks, f), dtype=np.int64),
                                      np.asarray(k["arrays"][f], dtype=np.int64)), (k["name"], f)
            assert ks.n_units == k["n_units"]
            assert ks.lines == k["lines"]
            assert list(ks.prefix_diagnostics) == k["diags"]
            assert meta["mnemonics"] == k["mnemonics"]
            assert meta["src_locs"] == k["src_locs"]
    assert n_err >= 30
