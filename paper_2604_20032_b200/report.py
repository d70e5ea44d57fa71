"""Stall reports assembled from the device outputs.

The device (libleo_b200 `leo_report`, csrc/report.cu) computes everything
data-dependent: single-dependency coverage before/after, the hotspot ranking,
each hotspot's cause order and its trace_chain.  This module turns those index
arrays into the reference's report objects (report.py:32-93) and renders them
in the reference's text and structured formats (report.py:221-346); the
output is byte-identical to `stalltrace.report.render_text` /
`render_structured` on the same inputs (tests/test_report.py against the
reference's corpus reports and generated fixtures).

Host metadata the device never sees (instruction text, offsets, source
locations, the latency-table echo) comes in a `ReportMeta`.
"""

from __future__ import annotations

import json
import sys
from dataclasses import dataclass, field, replace

import numpy as np

from . import diagnostics
from . import enums as E

CONSERVATION_REL_TOL = 1e-9          # report.py:29


# ---- report objects (mirrors of report.py:32-93; the reference's own classes
# are used instead when stalltrace is importable, see `classes()`) ----------

@dataclass(frozen=True)
class CauseReport:
    cause_offset: str | None
    mnemonic: str | None
    src_loc: str | None
    kind: str
    register: str | None
    blame_cycles: float
    pct: float
    factors: dict | None


@dataclass(frozen=True)
class ChainHopReport:
    offset: str
    mnemonic: str
    src_loc: str | None
    kind: str | None
    share_pct: float | None
    self_blame: str | None


@dataclass(frozen=True)
class HotspotReport:
    offset: str
    mnemonic: str
    src_loc: str | None
    stall_cycles: float
    share_pct: float
    breakdown: dict
    causes: tuple
    chain: tuple


@dataclass(frozen=True)
class CoverageReport:
    before: float
    after: float
    vacuous_before: bool
    vacuous_after: bool


@dataclass(frozen=True)
class ConfigEcho:
    stage_mask: tuple
    prune_exec: bool
    max_paths: int
    max_depth: int
    latency_units: str
    latency_table: dict


@dataclass(frozen=True)
class StallReport:
    kernel_name: str
    vendor: str
    period_cycles: int
    total_stall_cycles: float
    config: ConfigEcho
    coverage: CoverageReport
    hotspots: tuple
    diagnostics: tuple


class InternalInvariantError(RuntimeError):
    """errors.py:42-43 (analysis bug, not a user error)."""


def classes():
    """The report dataclasses to build: stalltrace's when importable."""
    try:
        from stalltrace import report as R
        return R
    except ImportError:
        return sys.modules[__name__]


@dataclass
class ReportMeta:
    """Host-side text of one kernel (disasm.py Instruction fields)."""
    kernel_name: str
    vendor: str
    period: int
    mnemonics: list
    src_locs: list                      # str(SourceLoc) or None per instruction
    echo: ConfigEcho
    prefix: tuple = field(default_factory=tuple)


def meta_from_reference(cfg, profile, config) -> ReportMeta:
    """ReportMeta of reference objects (KernelCfg, KernelProfile, AnalysisConfig)."""
    table = config.table_for(cfg.dialect)
    echo = ConfigEcho(stage_mask=tuple(config.stage_mask), prune_exec=config.prune_exec,
                      max_paths=config.max_paths, max_depth=config.max_depth,
                      latency_units=table.units,
                      latency_table={c.value: v for c, v in sorted(table.thresholds,
                                                                   key=lambda kv: kv[0].value)})
    ins = cfg.instructions
    return ReportMeta(kernel_name=cfg.kernel_name, vendor=cfg.dialect.value,
                      period=profile.sampling_period_cycles,
                      mnemonics=[i.mnemonic for i in ins],
                      src_locs=[str(i.src_loc) if i.src_loc else None for i in ins], echo=echo)


def _hex(off: int) -> str:
    return f"0x{off:04x}"


def _coverage(nodes: int, qualified: int) -> tuple[float, bool]:
    """single_dep_coverage's value / vacuous pair (analysis.py:553-561)."""
    if nodes == 0:
        return 1.0, True
    return qualified / nodes, False


def check_conservation(lat, period, e_stalled, e_blame):
    """Per stalled instruction, blame sums to S_j (report.py:145-155)."""
    if len(e_stalled) == 0:
        return
    if np.any(e_blame < 0):
        j = int(e_stalled[np.flatnonzero(e_blame < 0)[0]])
        raise InternalInvariantError(f"negative blame at index {j}")
    tot = np.zeros(len(lat), dtype=np.float64)
    np.add.at(tot, e_stalled, e_blame)
    s = lat.astype(np.float64) * float(period)
    js = np.unique(e_stalled)
    bad = np.abs(tot[js] - s[js]) > CONSERVATION_REL_TOL * np.maximum(np.abs(s[js]), 1.0)
    if np.any(bad):
        j = int(js[np.flatnonzero(bad)[0]])
        raise InternalInvariantError(f"blame conservation violated at index {j}: {tot[j]} != {s[j]}")


def assemble(ks, meta: ReportMeta, r: dict, rep: dict, diags: tuple, R=None):
    """StallReport from the device analysis `r` (device.Analyzer.result) and
    the device report arrays `rep` (device.Analyzer.report)."""
    R = R or classes()
    lat, cls_cnt, period = r["lat"], r["cls_cnt"], meta.period
    st, ed, sub, bl, fac = r["e_stalled"], r["e_edge"], r["e_sub"], r["e_blame"], r["e_factors"]
    pprod, pmeta = r["pprod"], r["pmeta"].astype(np.uint32)
    check_conservation(lat, period, st, bl)
    offs, mn, loc = ks.offset, meta.mnemonics, meta.src_locs
    S = lat.astype(np.int64) * int(period)
    total = float(S.sum())

    def s_at(i):
        return float(S[i])

    def cause_of(x):
        e = int(ed[x])
        return None if e < 0 else int(pprod[e])

    def kind_of(x):
        e = int(ed[x])
        return E.SELF_BLAMES[int(sub[x])] if e < 0 else E.EDGE_KINDS[(int(pmeta[e]) >> 27) & 7]

    def register_of(x):
        m = int(pmeta[int(ed[x])])
        return diagnostics.format_ref27(ks.dialect, m & 0x07FFFFFF) if ((m >> 27) & 7) < 2 else None

    hot = []
    for h in range(int(rep["n_hot"])):
        j = int(rep["hot"][h])
        s_j = s_at(j)
        causes = []
        for x in rep["causes"][h][:int(rep["n_causes"][h])]:
            x = int(x)
            b = float(bl[x])
            pct = (b / s_j * 100.0) if s_j else 0.0
            c = cause_of(x)
            if c is None:
                causes.append(R.CauseReport(cause_offset=None, mnemonic=None, src_loc=None,
                                            kind=kind_of(x), register=None, blame_cycles=b,
                                            pct=pct, factors=None))
            else:
                f = fac[x]
                causes.append(R.CauseReport(cause_offset=_hex(int(offs[c])), mnemonic=mn[c],
                                            src_loc=loc[c], kind=kind_of(x),
                                            register=register_of(x), blame_cycles=b, pct=pct,
                                            factors={"dist": float(f[0]), "eff": float(f[1]),
                                                     "isu": float(f[2]), "match": float(f[3])}))
        chain = []
        prev = None
        for t in range(int(rep["chain_len"][h])):
            node = int(rep["chain_node"][h][t])
            x = int(rep["chain_entry"][h][t])
            if x < 0:
                kind = share = None
            else:
                kind = kind_of(x)
                s_prev = s_at(prev)
                share = (float(bl[x]) / s_prev) if s_prev else None
            chain.append(R.ChainHopReport(offset=_hex(int(offs[node])), mnemonic=mn[node],
                                          src_loc=loc[node], kind=kind,
                                          share_pct=(share * 100.0) if share is not None else None,
                                          self_blame=None))
            prev = node
        if chain and int(rep["chain_self"][h]) >= 0:
            chain[-1] = replace(chain[-1], self_blame=kind_of(int(rep["chain_self"][h])))
        row = cls_cnt[j]
        breakdown = {name: int(row[k]) for name, k in
                     sorted((E.COMMON_STALLS[k], k) for k in range(len(E.COMMON_STALLS)))
                     if int(row[k]) > 0}
        hot.append(R.HotspotReport(offset=_hex(int(offs[j])), mnemonic=mn[j], src_loc=loc[j],
                                   stall_cycles=s_j,
                                   share_pct=(s_j / total * 100.0) if total else 0.0,
                                   breakdown=breakdown, causes=tuple(causes), chain=tuple(chain)))
    cov = rep["coverage"]
    before, vb = _coverage(int(cov[0]), int(cov[1]))
    after, va = _coverage(int(cov[2]), int(cov[3]))
    echo = meta.echo
    if R is not None and getattr(R, "ConfigEcho", None) is not ConfigEcho:
        echo = R.ConfigEcho(**{k: getattr(echo, k) for k in ("stage_mask", "prune_exec", "max_paths",
                                                             "max_depth", "latency_units",
                                                             "latency_table")})
    return R.StallReport(kernel_name=meta.kernel_name, vendor=meta.vendor, period_cycles=period,
                         total_stall_cycles=total, config=echo,
                         coverage=R.CoverageReport(before=before, after=after, vacuous_before=vb,
                                                   vacuous_after=va),
                         hotspots=tuple(hot), diagnostics=tuple(diags))


# ---- rendering (formats of report.py:221-346) -------------------------------

def _cycles(v: float) -> str:
    return f"{int(v)}" if v == int(v) else f"{v:.1f}"


def _header(rep) -> list[str]:
    cfg, cov = rep.config, rep.coverage
    stages = ",".join(map(str, cfg.stage_mask)) or "none"
    table = " ".join(f"{k}={_cycles(v)}" for k, v in cfg.latency_table.items())
    cov_txt = ["n/a (no edges)" if vac else f"{val:.3f}"
               for val, vac in ((cov.before, cov.vacuous_before), (cov.after, cov.vacuous_after))]
    return [
        f"kernel {rep.kernel_name} ({rep.vendor})",
        f"  total stall cycles: {_cycles(rep.total_stall_cycles)}  (sampling period "
        f"{rep.period_cycles} cycles)",
        f"  stages: {stages}  prune-exec: {'on' if cfg.prune_exec else 'off'}  path caps: "
        f"{cfg.max_paths} paths / {cfg.max_depth} deep",
        f"  latency thresholds ({cfg.latency_units}): {table}",
        f"  single-dependency coverage: before={cov_txt[0]} after={cov_txt[1]}",
        "",
    ]


def _cause_line(c) -> str:
    if c.cause_offset is None:
        return f"   {c.pct:5.1f}%  self ({c.kind})"
    reg = f" {c.register}" if c.register else ""
    where = f" ({c.src_loc})" if c.src_loc else ""
    return f"   {c.pct:5.1f}%  {c.kind}{reg} from {c.cause_offset} {c.mnemonic}{where}"


def _hop_line(hop) -> str:
    where = f" -- {hop.src_loc}" if hop.src_loc else ""
    if hop.kind is None:
        lead, tag = "     ", ""
    else:
        lead = "   ^ "
        pct = f" ({hop.share_pct:.1f}%)" if hop.share_pct is not None else ""
        tag = f"  [{hop.kind}{pct}]"
    note = f"  => self: {hop.self_blame}" if hop.self_blame else ""
    return f"{lead}{hop.offset} {hop.mnemonic}{where}{tag}{note}"


def _hotspot_lines(rank: int, spot) -> list[str]:
    where = f"  ({spot.src_loc})" if spot.src_loc else ""
    out = [f"#{rank} {spot.offset} {spot.mnemonic}{where}",
           f"   stall cycles: {_cycles(spot.stall_cycles)} ({spot.share_pct:.1f}% of kernel)"]
    if spot.breakdown:
        out.append("   stall breakdown: " + " ".join(f"{k}={v}" for k, v in spot.breakdown.items()))
    out.extend(_cause_line(c) for c in spot.causes)
    if len(spot.chain) > 1 or (spot.chain and spot.chain[0].self_blame):
        out.append("   chain:")
        out.extend(_hop_line(h) for h in spot.chain)
    out.append("")
    return out


def render_text(rep) -> str:
    """Text report, byte-identical to stalltrace.report.render_text."""
    lines = _header(rep)
    if not rep.hotspots:
        lines.append("  no samples")
    for rank, spot in enumerate(rep.hotspots, start=1):
        lines.extend(_hotspot_lines(rank, spot))
    if rep.diagnostics:
        lines.append("diagnostics:")
        lines.extend(f"  - {d}" for d in rep.diagnostics)
        lines.append("")
    return "\n".join(lines)


def _as_obj(rep) -> dict:
    cfg, cov = rep.config, rep.coverage

    def cause(c):
        return {"cause_offset": c.cause_offset, "mnemonic": c.mnemonic, "src_loc": c.src_loc,
                "kind": c.kind, "register": c.register, "blame_cycles": c.blame_cycles,
                "pct": c.pct, "factors": c.factors}

    def hop(h):
        return {"offset": h.offset, "mnemonic": h.mnemonic, "src_loc": h.src_loc, "kind": h.kind,
                "share_pct": h.share_pct, "self_blame": h.self_blame}

    return {
        "kernel": rep.kernel_name, "vendor": rep.vendor, "period_cycles": rep.period_cycles,
        "total_stall_cycles": rep.total_stall_cycles,
        "config": {"stage_mask": list(cfg.stage_mask), "prune_exec": cfg.prune_exec,
                   "max_paths": cfg.max_paths, "max_depth": cfg.max_depth,
                   "latency_units": cfg.latency_units, "latency_table": cfg.latency_table},
        "coverage": {"before": cov.before, "after": cov.after,
                     "vacuous_before": cov.vacuous_before, "vacuous_after": cov.vacuous_after},
        "hotspots": [{"offset": s.offset, "mnemonic": s.mnemonic, "src_loc": s.src_loc,
                      "stall_cycles": s.stall_cycles, "share_pct": s.share_pct,
                      "breakdown": s.breakdown, "causes": [cause(c) for c in s.causes],
                      "chain": [hop(h) for h in s.chain]} for s in rep.hotspots],
        "diagnostics": list(rep.diagnostics),
    }


def render_structured(reports) -> str:
    """JSON report(s), byte-identical to stalltrace.report.render_structured."""
    obj = [_as_obj(r) for r in reports] if isinstance(reports, (list, tuple)) else _as_obj(reports)
    return json.dumps(obj, indent=2) + "\n"


def parse_structured(text: str, R=None):
    """Report object(s) from the structured rendering (report.py:349-393)."""
    R = R or sys.modules[__name__]

    def one(o):
        cfg, cov = o["config"], o["coverage"]
        spots = tuple(
            R.HotspotReport(
                offset=h["offset"], mnemonic=h["mnemonic"], src_loc=h["src_loc"],
                stall_cycles=h["stall_cycles"], share_pct=h["share_pct"], breakdown=h["breakdown"],
                causes=tuple(R.CauseReport(**c) for c in h["causes"]),
                chain=tuple(R.ChainHopReport(**hop) for hop in h["chain"]))
            for h in o["hotspots"])
        return R.StallReport(
            kernel_name=o["kernel"], vendor=o["vendor"], period_cycles=o["period_cycles"],
            total_stall_cycles=o["total_stall_cycles"],
            config=R.ConfigEcho(stage_mask=tuple(cfg["stage_mask"]), prune_exec=cfg["prune_exec"],
                                max_paths=cfg["max_paths"], max_depth=cfg["max_depth"],
                                latency_units=cfg["latency_units"],
                                latency_table=cfg["latency_table"]),
            coverage=R.CoverageReport(**cov), hotspots=spots, diagnostics=tuple(o["diagnostics"]))

    obj = json.loads(text)
    return [one(o) for o in obj] if isinstance(obj, list) else one(obj)


def meta_from_fixture(rmeta: dict, mnemonics, srclocs, none: str = "\x00") -> ReportMeta:
    """ReportMeta of a golden report case (tests/golden/make_reports.py; numpy
    string arrays drop the NUL sentinel of a missing source location)."""
    e = rmeta["echo"]
    echo = ConfigEcho(stage_mask=tuple(e["stage_mask"]), prune_exec=e["prune_exec"],
                      max_paths=e["max_paths"], max_depth=e["max_depth"],
                      latency_units=e["latency_units"],
                      latency_table={k: v for k, v in e["latency_table"]})
    return ReportMeta(kernel_name=rmeta["kernel_name"], vendor=rmeta["vendor"], period=rmeta["period"],
                      mnemonics=[str(m) for m in mnemonics],
                      src_locs=[None if str(s) in ("", none) else str(s) for s in srclocs],
                      echo=echo)
