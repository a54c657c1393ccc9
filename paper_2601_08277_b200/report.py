"""Run reports in the reference's schema (proj/include/pic/report.hpp:23-103),
so the reference's tooling reads GPU results unchanged.

report_csv: header `csv_header()`, one row per step with doubles as %.17g,
then a summary row (totals of the timing columns, means of throughput and
moved fraction, counts of rebuilds and fired global sorts).
report_json: the same records under "steps" and "summary"; serialised like
nlohmann::json::dump() (keys sorted, no whitespace).
"""
from __future__ import annotations

import json

CSV_HEADER = ("step,wall_s,preproc_s,compute_s,sort_s,reduce_s,pps,fraction_moved,rebuilds,"
              "global_sort_reason")


def _g(v: float) -> str:
    return "%.17g" % v


def summarize(steps) -> dict:  # report.hpp:28-47
    s = dict(wall=0.0, preproc=0.0, compute=0.0, sort=0.0, reduce=0.0, mean_pps=0.0, mean_fraction=0.0,
             rebuilds=0, global_sorts=0)
    for m in steps:
        s["wall"] += m.wall_s
        s["preproc"] += m.preproc_s
        s["compute"] += m.compute_s
        s["sort"] += m.sort_s
        s["reduce"] += m.reduce_s
        s["mean_pps"] += m.particles_per_second
        s["mean_fraction"] += m.fraction_moved
        s["rebuilds"] += int(m.rebuilds)
        s["global_sorts"] += m.global_sort != "none"
    if steps:
        s["mean_pps"] /= len(steps)
        s["mean_fraction"] /= len(steps)
    return s


def report_csv(steps) -> str:  # report.hpp:55-73
    out = CSV_HEADER + "\n"
    if not steps:
        return out
    for m in steps:
        out += ",".join([str(m.step), _g(m.wall_s), _g(m.preproc_s), _g(m.compute_s), _g(m.sort_s), _g(m.reduce_s),
                         _g(m.particles_per_second), _g(m.fraction_moved), str(int(m.rebuilds)), m.global_sort]) + "\n"
    s = summarize(steps)
    out += ",".join(["summary", _g(s["wall"]), _g(s["preproc"]), _g(s["compute"]), _g(s["sort"]), _g(s["reduce"]),
                     _g(s["mean_pps"]), _g(s["mean_fraction"]), str(s["rebuilds"]), str(s["global_sorts"])]) + "\n"
    return out


def report_json(steps) -> dict:  # report.hpp:76-103
    j = {"steps": []}
    if not steps:
        return j
    for m in steps:
        j["steps"].append({"step": int(m.step), "wall_s": m.wall_s, "preproc_s": m.preproc_s,
                           "compute_s": m.compute_s, "sort_s": m.sort_s, "reduce_s": m.reduce_s,
                           "pps": m.particles_per_second, "fraction_moved": m.fraction_moved,
                           "rebuilds": int(m.rebuilds), "global_sort_reason": m.global_sort})
    s = summarize(steps)
    j["summary"] = {"wall_s": s["wall"], "preproc_s": s["preproc"], "compute_s": s["compute"], "sort_s": s["sort"],
                    "reduce_s": s["reduce"], "mean_pps": s["mean_pps"], "mean_fraction_moved": s["mean_fraction"],
                    "rebuilds": s["rebuilds"], "global_sorts": s["global_sorts"]}
    return j


def dump_json(j: dict) -> str:
    """nlohmann::json::dump() layout: object keys sorted, no whitespace."""
    return json.dumps(j, sort_keys=True, separators=(",", ":"))
