"""Batching independent kernels into one pipeline pass (paper_2604_20032_b200.batch):
the oracle on the concatenation, split per kernel, equals the oracle on each
kernel alone — edges, pruned edges, paths, diagnostics, blame, slice."""

import numpy as np

import parity
from oracle import oracle
from paper_2604_20032_b200 import batch as BT
from paper_2604_20032_b200 import synth


def _wls(dialect, n, seeds):
    lines = synth.LineTable(32, seed=999)
    return [synth.make_workload(dialect, n, 20 * n, s, lines=lines, name=f"k{s}") for s in seeds]


def _oracle_dict(ks, r):
    return dict(bprod=r.prod, bcons=r.cons, bmeta=r.meta, pprod=r.p_prod, pcons=r.p_cons,
                pmeta=r.p_meta, npaths=r.p_npaths, first=r.p_first, plen=r.path_len,
                pacc=r.path_acc, e_stalled=r.e_stalled, e_edge=r.e_edge, e_sub=r.e_sub,
                e_blame=r.e_blame, e_factors=r.e_factors, level=r.level, diag_records=r.diags,
                n_regular=r.n_regular, p_n_regular=int(np.sum(((r.p_meta >> 27) & 7) < 2)))


def test_batch_split_equals_per_kernel_oracle():
    for dialect in ("amd", "nvidia", "intel"):
        wls = _wls(dialect, 300, range(5))
        b = BT.concat(wls)
        rb = oracle.run(b.kernel, synth.bin_host(b))
        parts = BT.split_result(b, _oracle_dict(b.kernel, rb))
        for wl, got in zip(wls, parts):
            r = oracle.run(wl.kernel, synth.bin_host(wl))
            exp = _oracle_dict(wl.kernel, r)
            for f in ("bprod", "bcons", "bmeta", "pprod", "pcons", "pmeta", "npaths", "e_stalled",
                      "e_edge", "e_sub", "e_blame", "e_factors", "level"):
                assert np.array_equal(exp[f], got[f]), (dialect, wl.kernel.name, f)
            for x in range(len(exp["pprod"])):
                assert parity._paths(exp, x) == parity._paths(got, x)
            assert sorted(map(tuple, exp["diag_records"][:, :5].tolist())) == \
                sorted(map(tuple, got["diag_records"][:, :5].tolist()))
