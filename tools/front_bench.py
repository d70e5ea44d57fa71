"""Listing -> SoA throughput: native front-end vs the reference's
parse_kernels + soa.encode_cfg (run where `stalltrace` is importable).

    python tools/front_bench.py [n_instr]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), "/root/reference/pkg/src"]
import stalltrace as st  # noqa: E402
from stalltrace import disasm  # noqa: E402

from paper_2604_20032_b200 import front, soa, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
for d in ("nvidia", "amd", "intel"):
    wl = synth.make_workload(d, n, 10, seed=5)
    cfg = soa.decode_to_reference(wl.kernel, None, st)
    text = disasm.format_listing("k", list(cfg.instructions))
    table = front.default_table_text(d)
    t0 = time.perf_counter()
    got = front.parse_kernels_soa(d, text, table)
    t1 = time.perf_counter()
    ref = {k: soa.encode_cfg(v) for k, v in disasm.parse_kernels(st.Dialect(d), text).items()}
    t2 = time.perf_counter()
    same = all((getattr(got["k"][0], f) == getattr(ref["k"], f)).all() for f in ("opnd", "succ", "pred"))
    print(f"{d}: {n} instrs, {len(text) / 1e6:.1f} MB  native {1e3 * (t1 - t0):.1f} ms  "
          f"reference {1e3 * (t2 - t1):.1f} ms  ({(t2 - t1) / (t1 - t0):.0f}x)  same={same}")
