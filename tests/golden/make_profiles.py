"""Golden vectors for the native profile loader (native/leo_profile.cpp).

Runs the REFERENCE's `profile.load_profiles` / `attach` (profile.py:186-366)
in this container (needs /root/reference/pkg/src importable) on:
  * the three corpus `.prof` files, attached to the corpus listings
    (expected = soa.encode_profile(attach(cfg, prof)) + attach diagnostics);
  * valid random documents (every field kind, vendor-category spelling
    variants, hex offset spellings, JSON Lines and pretty-printed);
  * seeded mutations of those: byte-level edits (malformed JSON) and
    field-level edits (every ProfileError / InputError the schema raises).
Cases where the reference fails with something other than ProfileError /
InputError (a TypeError on a non-numeric stall count, ...) or uses a value the
SoA cannot hold are not recorded (leo_profile.cpp's header lists them).

    python tests/golden/make_profiles.py      # -> tests/golden/profiles.json.gz
"""

from __future__ import annotations

import gzip
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(ROOT)]

from stalltrace import disasm, profile  # noqa: E402
from stalltrace.errors import InputError, ProfileError  # noqa: E402
from stalltrace.isa import Dialect  # noqa: E402

from paper_2604_20032_b200 import soa  # noqa: E402

CATS = {d.value: sorted(profile._STALL_MAPS[d]) for d in Dialect}
WEIRD = [None, True, False, 0, -1, 1, 7, 2 ** 40, 1.5, -0.0, 1e300, 0.5, 1e-5, "x", "0x10", "",
         [], [1, "a"], {}, {"a": 1}, "éß", 3.0, 1e16, 12345678.9]


def spell(cat: str, rng: random.Random) -> str:
    r = rng.random()
    if r < 0.2:
        return cat.upper()
    if r < 0.3:
        return "  " + cat.replace(" ", "   ").title() + " "
    if r < 0.35:
        return cat.replace(" ", "\t")
    return cat


def offset_spelling(off: int, rng: random.Random):
    r = rng.random()
    if r < 0.1:
        return off
    if r < 0.2:
        return f"0X{off:X}"
    if r < 0.25:
        return f" 0x{off:x} "
    if r < 0.3:
        return f"{off:x}"
    if r < 0.33:
        return f"+0x{off:x}"
    if r < 0.36 and off >= 16:
        h = f"{off:x}"
        return "0x" + h[0] + "_" + h[1:]
    if r < 0.38:
        return f"0x_{off:x}"
    return f"0x{off:x}"


def random_record(dialect: str, off, rng: random.Random) -> dict:
    cats = rng.sample(CATS[dialect], rng.randint(0, min(4, len(CATS[dialect]))))
    counts = {spell(c, rng): rng.randint(0, 9) for c in cats}
    lat = sum(counts.values())
    rec = {"offset": off, "counts": counts, "latency_samples": lat}
    if rng.random() < 0.5:
        rec["total_samples"] = lat + rng.randint(0, 5)
    if rng.random() < 0.5:
        rec["exec_count"] = rng.randint(0, 5000)
    if rng.random() < 0.5:
        rec["efficiency"] = rng.choice([1, 1.0, 0.5, 0.25, 0.125, 1e-3, rng.random() or 0.5])
    if rng.random() < 0.1:
        rec["total_samples"] = None
    return rec


def random_doc(rng: random.Random, n_kernels: int | None = None) -> tuple[str, list]:
    objs = []
    for k in range(n_kernels or rng.randint(1, 3)):
        dialect = rng.choice(list(CATS))
        offs = rng.sample(range(0, 4096, rng.choice([4, 8, 16])), rng.randint(0, 12))
        obj = {"kernel": rng.choice([f"k{k}", f"kernel_{k}", f"_Z{k}fooPf", f"ké{k}"]),
               "vendor": rng.choice([dialect, dialect.upper(), f" {dialect} "]),
               "period_cycles": rng.choice([1, 64, 100, 4096]),
               "samples": [random_record(dialect, offset_spelling(o, rng), rng) for o in offs]}
        keys = list(obj)
        rng.shuffle(keys)
        objs.append({key: obj[key] for key in keys})
    sep = rng.choice(["\n", "\n\n", " ", "\r\n"])
    indent = rng.choice([None, None, 2])
    text = sep.join(json.dumps(o, indent=indent, ensure_ascii=rng.random() < 0.5) for o in objs)
    return text + rng.choice(["", "\n", "  \n"]), objs


def semantic_mutation(objs: list, rng: random.Random) -> str:
    objs = json.loads(json.dumps(objs))
    o = rng.choice(objs)
    r = rng.randrange(20)
    recs = o["samples"]
    if r == 0:
        o.pop(rng.choice(["kernel", "vendor", "period_cycles", "samples"]))
    elif r == 1:
        o[rng.choice(["extra", "Zeta", "alpha"])] = 1
    elif r == 2:
        o["vendor"] = rng.choice(["arm", "", 5, None, "nvidia2", "Intel ", ["amd"]])
    elif r == 3:
        o["period_cycles"] = rng.choice(WEIRD)
    elif r == 4:
        o["samples"] = rng.choice(WEIRD)
    elif r == 5:
        o["kernel"] = rng.choice(WEIRD + [objs[0]["kernel"]])
    elif recs:
        rec = rng.choice(recs)
        if r == 6:
            rec.pop(rng.choice(["offset", "counts", "latency_samples"]))
        elif r == 7:
            rec[rng.choice(["bogus", "Offset", "a_field"])] = 0
        elif r == 8:
            rec["offset"] = rng.choice(WEIRD + ["0xg", "0x", "1__0", "_10", "10_", "-0x5", "0x-5",
                                                " 0x1f\t", "0b11", "ff", "FF"])
        elif r == 9:
            rec["counts"] = rng.choice(WEIRD)
        elif r == 10:
            rec["counts"][rng.choice(["quantum flux", "Memory", "sleeping", "pipestall", "other"])] = 1
        elif r == 11:
            rec["latency_samples"] = rng.choice(WEIRD + [rec["latency_samples"] + 1])
        elif r == 12:
            rec["total_samples"] = rng.choice(WEIRD + [0])
        elif r == 13:
            rec["exec_count"] = rng.choice(WEIRD)
        elif r == 14:
            rec["efficiency"] = rng.choice(WEIRD + [0.0, 1.0000001, 2, 5e-324, "1"])
        elif r == 15 and rec["counts"]:
            key = rng.choice(list(rec["counts"]))
            rec["counts"][key] = rng.choice([-1, 0, 3, True])
        elif r == 16:
            recs.append(dict(rec))
        elif r == 17:
            rng.choice(objs)["samples"] = [rng.choice(WEIRD)]
        else:
            return json.dumps(objs[0]) + "\n" + json.dumps(objs[0])   # duplicate kernel entries
    return "\n".join(json.dumps(x, ensure_ascii=False) for x in objs)


def byte_mutation(text: str, rng: random.Random) -> str:
    t = list(text)
    for _ in range(rng.randint(1, 2)):
        if not t:
            break
        r = rng.randrange(6)
        i = rng.randrange(len(t))
        if r == 0:
            del t[i]
        elif r == 1:
            t.insert(i, rng.choice(list('{}[]:,"\\ \n\tx0-.eE') + ["\x01", "é", "NaN", "true",
                                                                     "\\u12", "\\ud83d\\ude00"]))
        elif r == 2:
            t[i] = rng.choice(list('{}[]:,"\\'))
        elif r == 3:
            del t[i:]
        elif r == 4:
            t.insert(i, rng.choice(["Infinity", "-Infinity", "1e400", "-", "01", "1.", ".5", "null"]))
        else:
            t[i:i] = t[max(0, i - 5):i]
    return "".join(t)


def reference_outcome(text: str):
    """('ok', kernels) | ('ProfileError'|'InputError', message) | None (skipped)."""
    try:
        profs = profile.load_profiles(text)
    except (ProfileError, InputError) as exc:
        return [type(exc).__name__ if isinstance(exc, ProfileError) else "InputError", str(exc)]
    except Exception:
        return None
    smap = profile._STALL_MAPS
    kernels = []
    for p in profs:
        recs = []
        for s in p.samples:
            cls = [0] * 8
            for c, v in s.vendor_counts:
                if type(v) is not int and type(v) is not bool:
                    return None
                cls[list(profile.CommonStall).index(smap[p.dialect][profile._norm(c)])] += int(v)
            if not (-2 ** 63 <= s.offset < 2 ** 63) or s.latency_samples >= 2 ** 31 \
                    or (s.exec_count or 0) >= 2 ** 63 or (s.total_samples or 0) >= 2 ** 31:
                return None
            recs.append([s.offset, int(s.latency_samples),
                         -1 if s.total_samples is None else int(s.total_samples),
                         -1 if s.exec_count is None else int(s.exec_count),
                         float(s.efficiency).hex(), cls])
        if not (0 < p.sampling_period_cycles < 2 ** 63):
            return None
        kernels.append([p.kernel_name, p.dialect.value, int(p.sampling_period_cycles), recs])
    return ["ok", kernels]


def corpus_cases() -> list:
    out = []
    for d in ("nvidia", "amd", "intel"):
        listing = (REF / "tests" / "corpus" / f"ltimes_{d}.s").read_text()
        text = (REF / "tests" / "corpus" / f"ltimes_{d}.prof").read_text()
        cfgs = disasm.parse_kernels(Dialect(d), listing)
        profs = {p.kernel_name: p for p in profile.load_profiles(text)}
        for name, cfg in sorted(cfgs.items()):
            att = profile.attach(cfg, profs[name])
            ps = soa.encode_profile(att)
            table = (REF / "src" / "stalltrace" / "data" / f"{d}.opcodes").read_text()
            out.append(dict(dialect=d, listing=listing, table=table, profile=text, kernel=name,
                            period=ps.period, lat=ps.lat.tolist(), cls_cnt=ps.cls_cnt.tolist(),
                            exec_cnt=ps.exec_cnt.tolist(), total=ps.total.tolist(),
                            eff=[float(x).hex() for x in ps.eff], sampled=ps.sampled.tolist(),
                            diagnostics=list(att.diagnostics)))
    return out


def main():
    rng = random.Random(20260417)
    cases, seen = [], set()

    def add(text):
        if text in seen:
            return
        exp = reference_outcome(text)
        if exp is None:
            return
        seen.add(text)
        cases.append([text, exp])

    for f in sorted((REF / "tests" / "corpus").glob("*.prof")):
        add(f.read_text())
    for text in ["", "   \n", "[]", "{}", "null", '{"kernel": "k"}', "1 2", "{\"a\":1}{",
                 '{"kernel":"k","vendor":"amd","period_cycles":1,"samples":[]}  ',
                 '{"kernel":"k","vendor":"amd","period_cycles":1,"samples":[]} x']:
        add(text)
    for _ in range(700):
        text, objs = random_doc(rng)
        add(text)
        add(semantic_mutation(objs, rng))
        add(semantic_mutation(objs, rng))
        add(byte_mutation(text, rng))
    kinds = {}
    for _, e in cases:
        key = e[0] if e[0] == "ok" else e[1].split(":")[0][:40]
        kinds[key] = kinds.get(key, 0) + 1
    doc = dict(cases=cases, corpus=corpus_cases())
    with gzip.open(HERE / "profiles.json.gz", "wt", encoding="utf-8") as f:
        json.dump(doc, f, ensure_ascii=False, separators=(",", ":"))
    print(f"{len(cases)} documents; outcomes:")
    for k, v in sorted(kinds.items(), key=lambda kv: -kv[1]):
        print(f"  {v:5d}  {k}")


if __name__ == "__main__":
    main()
