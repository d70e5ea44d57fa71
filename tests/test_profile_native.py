"""Native profile loader (native/leo_profile.cpp, front.ProfileDoc) against the
reference's load_profiles / attach (profile.py:186-366), through golden
vectors made by running the reference (tests/golden/make_profiles.py):
every accepted document's records, every rejected document's exact
ProfileError / InputError text, and the corpus profiles attached to the
corpus listings (ProfileSoA + skid diagnostics).  CPU only."""

import gzip
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2604_20032_b200 import front

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def golden():
    with gzip.open(GOLDEN / "profiles.json.gz", "rt", encoding="utf-8") as f:
        return json.load(f)


def outcome(text):
    try:
        doc = front.load_profiles(text)
    except front.ProfileError as exc:
        return ["ProfileError", str(exc)]
    except front.InputError as exc:
        return ["InputError", str(exc)]
    kernels = []
    for k, (name, dialect, period, _n) in enumerate(doc.kernels):
        r = doc.records(k)
        recs = [[int(r["offset"][i]), int(r["lat"][i]), int(r["total"][i]), int(r["exec_cnt"][i]),
                 float(r["eff"][i]).hex(), r["cls_cnt"][i].tolist()] for i in range(len(r["offset"]))]
        kernels.append([name, dialect, period, recs])
    return ["ok", kernels]


def test_documents_match_reference(golden):
    bad = []
    for text, exp in golden["cases"]:
        got = outcome(text)
        if got != exp:
            bad.append((text[:120], exp if exp[0] != "ok" else "ok", got if got[0] != "ok" else "ok"))
    assert not bad, f"{len(bad)} of {len(golden['cases'])} differ, first: {bad[:3]}"
    kinds = {e[0] for _, e in golden["cases"]}
    assert kinds >= {"ok", "ProfileError", "InputError"}


def test_corpus_attach_matches_reference(golden):
    assert len(golden["corpus"]) == 3
    for c in golden["corpus"]:
        pairs = front.load_inputs(c["dialect"], c["listing"], c["profile"], c["table"], kernel=c["kernel"])
        (ks, prof), = pairs
        assert prof.period == c["period"]
        for key in ("lat", "cls_cnt", "exec_cnt", "total", "sampled"):
            assert np.array_equal(getattr(prof, key), np.array(c[key])), key
        assert [x.hex() for x in prof.eff] == c["eff"]
        assert ks.prefix_diagnostics[:len(c["diagnostics"])] == tuple(c["diagnostics"])


def test_attach_mismatch_and_skid():
    doc = front.load_profiles(
        '{"kernel": "k", "vendor": "amd", "period_cycles": 4, "samples": ['
        '{"offset": "0x4", "counts": {"ALU dependency": 3}, "latency_samples": 3},'
        '{"offset": "0x30", "counts": {}, "latency_samples": 0},'
        '{"offset": 16, "counts": {}, "latency_samples": 0}]}')
    from paper_2604_20032_b200.soa import KernelSoA
    n = 3
    ks = KernelSoA(name="k", dialect="amd", opclass=np.zeros(n, np.uint8), block_of=np.zeros(n, np.int32),
                   opnd_ptr=np.zeros(n + 1, np.int32), opnd=np.zeros(0, np.uint32),
                   sync_kind=np.zeros(n, np.uint8), sync_a=np.zeros(n, np.uint32),
                   sync_b=np.zeros(n, np.uint32), blk_first=np.zeros(1, np.int32),
                   blk_last=np.full(1, n - 1, np.int32), succ_ptr=np.zeros(2, np.int32),
                   succ=np.zeros(0, np.int32), pred_ptr=np.zeros(2, np.int32), pred=np.zeros(0, np.int32),
                   unit_base=np.zeros(8, np.int32), n_units=0, offset=np.array([0, 4, 8]),
                   line_id=np.zeros(n, np.int32), lines=["<unknown>"], prefix_diagnostics=())
    prof, diags = doc.attach(ks)
    assert prof.lat.tolist() == [0, 3, 0] and prof.sampled.tolist() == [0, 1, 0]
    assert prof.cls_cnt[1].tolist() == [0, 3, 0, 0, 0, 0, 0, 0]
    assert diags == ("2 sampled offset(s) match no instruction (skid): 0x10, 0x30",)
    ks.name = "other"
    with pytest.raises(front.ProfileError, match="profile kernel 'k' does not match disassembly kernel 'other'"):
        doc.attach(ks, 0)
    ks.name, ks.dialect = "k", "nvidia"
    with pytest.raises(front.ProfileError, match="profile vendor amd does not match disassembly dialect nvidia"):
        doc.attach(ks, 0)


def test_big_document_parallel_records_and_first_error():
    """> 16 K records take the multi-threaded record pass: records stay in
    document order, and with several bad records the error raised is the
    first one in document order (what the reference's sequential loop
    raises; message formats as pinned by the golden documents)."""
    import json as _json
    n = 40000
    cats = ["ALU dependency", "waiting for memory", "barrier wait"]
    recs = [{"offset": f"0x{4 * i:x}", "counts": {cats[i % 3]: i % 7, "other": 1},
             "latency_samples": i % 7 + 1, "exec_count": i} for i in range(n)]
    doc = {"kernel": "big", "vendor": "amd", "period_cycles": 64, "samples": recs}
    d = front.load_profiles(_json.dumps(doc))
    r = d.records(0)
    assert r["offset"].tolist() == [4 * i for i in range(n)]
    assert r["lat"].tolist() == [i % 7 + 1 for i in range(n)]
    assert r["exec_cnt"].tolist() == list(range(n))
    cls = r["cls_cnt"]
    # ALU dependency -> execution_dep (1), waiting for memory -> memory_dep (0),
    # barrier wait -> synchronization (2), other -> other (7)
    idx = {0: 1, 1: 0, 2: 2}
    for i in (0, 1, 2, 12345, n - 1):
        assert cls[i, idx[i % 3]] == i % 7 and cls[i, 7] == 1
    bad = _json.loads(_json.dumps(doc))
    bad["samples"][31000]["bogus"] = 1                     # later chunk
    bad["samples"][17003]["counts"]["other"] = -1          # earlier chunk: reported
    with pytest.raises(front.ProfileError, match=r"^negative stall count at offset 0x109ac$"):
        front.load_profiles(_json.dumps(bad))
    bad["samples"][5]["latency_samples"] = "x"             # earliest
    with pytest.raises(front.ProfileError, match=r"^latency_samples must be an integer at offset 0x14$"):
        front.load_profiles(_json.dumps(bad))
