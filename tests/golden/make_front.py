"""Generate tests/golden/front.npz by running the REFERENCE's listing front-end
(disasm.parse_kernels, disasm.py:259-626) here, flattened with soa.encode_cfg.

    python tests/golden/make_front.py

Listings: the bundled corpus, `format_listing` renderings of random_world
kernels (generators.py) and of decoded synthetic kernels, hand-written
edge cases (labels, guarded terminators, calls, inline stacks, missing
offsets, unreachable blocks) and a set of malformed listings whose
ListingError text the native parser must reproduce.  The three default
opcode tables (stalltrace/data/*.opcodes) are stored with the cases: the
native front-end takes the table text as input, like the reference's
`table` argument.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REPO), str(REF / "tests"), str(REPO / "tests"), str(REF / "src")]

import stalltrace as st  # noqa: E402
from stalltrace import disasm  # noqa: E402
from stalltrace.errors import ListingError  # noqa: E402

from paper_2604_20032_b200 import soa, synth  # noqa: E402

OUT = REPO / "tests" / "golden" / "front.npz"
K_FIELDS = ("opclass", "block_of", "opnd_ptr", "opnd", "sync_kind", "sync_a", "sync_b", "blk_first",
            "blk_last", "succ_ptr", "succ", "pred_ptr", "pred", "unit_base", "offset", "line_id")

EDGE = {
    "nvidia": [
        ".kernel k\n/*0010*/ @P0 DFMA R4, R2, R6, R4 {wait=B1 write=B2 stall=4} // LTimes.cpp:62\n",
        ".kernel k\n@!P3 MOV R0, R1\nIADD3 R0, R1, R2 // a.cpp:10 <- b.hpp:20 <- c.hpp:30\nEXIT\n",
        ".kernel k\nMOV R0, R1 // not a location\nDEPBAR {depbar=B2,B4}\nUMOV UR4, UR5\nLDG.E.128 R8, R2\n"
        "ATOMG.E.64 R10, R2, R4\nEXIT\n",
        ".kernel a\nL0:\n  MOV R0, R1\n@P1 BRA L0\nCALL.REL fn\nfn:\nRET\n.kernel b\n@P0 EXIT\nMOV R1, R2\n",
        ".kernel k\nBRA L1\nMOV R0, R1\nL1:\nEXIT\nMOV R2, R3\n",
        ".kernel k\n/*00a0*/ MOV R0, 0x10\n\n# comment\n// full line\n/*00b0*/ ST.E [R2], R0\nFADD R1, R2, -3\n",
        ".kernel k\n  IADD3 R0, R1, R2   // f.cu:007\nBAR.SYNC 0x0 {read=B3}\nEXIT // g.cu:1 <- h.cu:x\n",
        ".kernel k\nMOV R0 , R1,R2\r\nEXIT\r\n",
        ".kernel k\n@P2 BRA.U L0\nMOV R0, R1 {}\nL0:\nEXIT\n",
    ],
    "amd": [
        ".kernel k\ns_waitcnt vmcnt(0) lgkmcnt(0)\nglobal_load_dwordx2 v[6:7], v[4:5], off\n"
        "global_store_dword v[0:1], v2\ns_endpgm\n",
        ".kernel k\nBB0:\ns_cbranch_scc1 BB1\nv_add_f32 v0, v1, v2 // x.cpp:3\nBB1:\ns_waitcnt lgkmcnt(3)\n"
        "s_load_dword s4, s[0:1], 0x10\ns_call_b64 s[2:3], foo\nfoo:\ns_endpgm\n",
        ".kernel k\nv_mov_b32 v0, P1\ns_branch BB2\nBB2:\nv_cmp_eq_u32 vcc, v0, v1\n",
    ],
    "intel": [
        ".kernel k\nsend.dc0 r10, r4 {sbid.set=5}\nadd r1:+1, r2, r3 {sbid.wait.dst=5 sbid.wait.src=1,2}\n"
        "@P0 goto L0\nL0:\neot\n",
        ".kernel k\nmov r0, r1\nL:\n@P1 while L\nret\n",
    ],
}

BAD = {
    "nvidia": [
        ".kernel k\nIADD3 R0, ???\n",
        ".kernel k\n/*0000*/ MOV R0, R1\n/*0000*/ MOV R2, R3\n",
        ".kernel k\n/*0010*/ MOV R0, R1\n/*0000*/ MOV R2, R3\n",
        ".kernel k\nLDG R0, R2 {write=B7}\n",
        ".kernel k\nMOV R0, R1 {sbid.set=3}\n",
        "MOV R0, R1\n",
        "L0:\n",
        ".kernel k\nBRA L9\nEXIT\n",
        ".kernel k\n@P7 MOV R0, R1\n",
        ".kernel k\nMOV R0, P9\n",
        ".kernel k\nMOV R0, B0\n",
        ".kernel k\nMOV R0, R1 {wait=X1}\n",
        ".kernel k\nMOV R0, R1 {stall=-1}\n",
        ".kernel k\nMOV R0, R1 {bogus}\n",
        ".kernel k\nMOV R0, R1 {foo=1}\n",
        ".kernel k\nMOV R0, R1 {wait=B1\n",
        ".kernel k\nMOV R0, R1 {wait=B1} junk\n",
        ".kernel k\nBRA L0, L1\nL0:\nL1:\nEXIT\n",
        ".kernel k\nMOV R0, R1\nL9:\n",
        ".kernel k\nL0:\nMOV R0, R1\nL0:\nEXIT\n",
        ".kernel k\n.kernel j\nEXIT\n",
        ".kernel k\nEXIT\n.kernel k\nEXIT\n",
        "# nothing\n",
        ".kernel k\n123 MOV\n",
        ".kernel k\nMOV R0, vmcnt(0)\n",
    ],
    "amd": [
        ".kernel k\nv_mov_b32 v0, v1 {wait=B1}\n",
        ".kernel k\nv_mov_b32 v[3:1], v1\n",
        ".kernel k\ns_waitcnt vmcnt(0) {x=1}\n",
        ".kernel k\ns_waitcnt vmcnt(x)\n",
    ],
    "intel": [
        ".kernel k\nsend r1, r2 {sbid.set=32}\n",
        ".kernel k\nadd r1, r2 {sbid.wait.dst=40}\n",
        ".kernel k\nadd r1, r2 {sbid.wait.src=a}\n",
        ".kernel k\nadd r1, r2 {stall=3}\n",
    ],
}


def tables():
    data = REF / "src" / "stalltrace" / "data"
    return {d: (data / f"{d}.opcodes").read_text() for d in ("nvidia", "amd", "intel")}


def main():
    import generators
    texts = []
    for d, ts in EDGE.items():
        texts += [(d, t) for t in ts]
    corpus = REF / "tests" / "corpus"
    for d in ("nvidia", "amd", "intel"):
        texts.append((d, (corpus / f"ltimes_{d}.s").read_text()))
        for s in range(40):
            att = generators.random_world(s, st.Dialect(d))
            texts.append((d, disasm.format_listing(att.cfg.kernel_name, list(att.cfg.instructions))))
        wl = synth.make_workload(d, 2000, 1000, seed=70 + len(d))
        cfg = soa.decode_to_reference(wl.kernel, None, st)
        texts.append((d, disasm.format_listing("synth", list(cfg.instructions))))
    for d, ts in BAD.items():
        texts += [(d, t) for t in ts]
    cases = []
    for d, text in texts:
        rec = {"dialect": d, "text": text}
        try:
            kernels = disasm.parse_kernels(st.Dialect(d), text)
        except ListingError as e:
            rec["error"] = str(e)
            cases.append(rec)
            continue
        out = []
        for name, cfg in kernels.items():
            ks = soa.encode_cfg(cfg)
            out.append({"name": name,
                        "arrays": {f: np.asarray(getattr(ks, f)).astype(np.int64).tolist() for f in K_FIELDS},
                        "n_units": ks.n_units, "lines": list(ks.lines), "diags": list(cfg.diagnostics),
                        "mnemonics": [i.mnemonic for i in cfg.instructions],
                        "src_locs": [str(i.src_loc) if i.src_loc else None for i in cfg.instructions]})
        rec["kernels"] = out
        cases.append(rec)
    np.savez_compressed(OUT, cases=np.array(json.dumps(cases)), tables=np.array(json.dumps(tables())))
    print("front cases:", len(cases), "errors:", sum("error" in c for c in cases))


if __name__ == "__main__":
    main()
