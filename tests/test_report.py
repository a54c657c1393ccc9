"""Run reports in the reference's schema (report.hpp:23-103): the Python and
the C++ writers (include/picgpu.hpp) agree byte for byte, and the summary row
follows the reference's rule (totals, means, counts)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

STEPS = [  # step, wall, preproc, compute, sort, reduce, pps, fraction, rebuilds, reason
    (0, 0.0125, 0.0, 0.00153, 0.00126, 0.0, 1.1656796094309586e10, 0.011918863654136658, 0, "none"),
    (1, 1e-05, 0.0, 2.5e-3, 1.0 / 3.0, 0.0, 123456789.0, 0.1, 1, "interval"),
    (2, 0.3, 0.0, 0.1, 0.2, 0.0, 7e-300, 0.0, 2, "slot_ratio"),
]


def _metrics(pg):
    return [pg.StepMetrics(s, w, p, c, so, r, pps, f, rb, reason) for s, w, p, c, so, r, pps, f, rb, reason in STEPS]


def test_csv_schema(pg):
    from paper_2601_08277_b200.report import CSV_HEADER, report_csv

    out = report_csv(_metrics(pg)).splitlines()
    assert out[0] == CSV_HEADER == ("step,wall_s,preproc_s,compute_s,sort_s,reduce_s,pps,fraction_moved,rebuilds,"
                                    "global_sort_reason")
    assert out[2].split(",")[1] == "1.0000000000000001e-05" and out[2].endswith(",1,interval")
    summ = out[-1].split(",")
    assert summ[0] == "summary" and summ[-2:] == ["3", "2"]  # rebuild count, fired sorts
    assert float(summ[1]) == pytest.approx(0.0125 + 1e-05 + 0.3)
    assert report_csv([]) == CSV_HEADER + "\n"


def test_json_schema(pg):
    from paper_2601_08277_b200.report import report_json

    j = report_json(_metrics(pg))
    assert set(j) == {"steps", "summary"} and len(j["steps"]) == 3
    assert set(j["steps"][0]) == {"step", "wall_s", "preproc_s", "compute_s", "sort_s", "reduce_s", "pps",
                                  "fraction_moved", "rebuilds", "global_sort_reason"}
    assert j["summary"]["global_sorts"] == 2 and j["summary"]["rebuilds"] == 3
    assert report_json([]) == {"steps": []}


def test_python_and_cpp_writers_agree(pg, tmp_path):
    from paper_2601_08277_b200.report import dump_json, report_csv, report_json

    reasons = {"none": "none", "interval": "interval", "rebuilds": "rebuilds", "slot_ratio": "slot_ratio"}
    rows = "\n".join(
        f"    {{ picgpu::StepMetrics m; m.step = {s}; m.wall_s = {w!r}; m.preproc_s = {p!r}; m.compute_s = {c!r};"
        f" m.sort_s = {so!r}; m.reduce_s = {r!r}; m.particles_per_second = {pps!r}; m.fraction_moved = {f!r};"
        f" m.rebuilds = {rb}; m.global_sort = picgpu::SortReason::{reasons[reason]}; v.push_back(m); }}"
        for s, w, p, c, so, r, pps, f, rb, reason in STEPS)
    src = tmp_path / "r.cpp"
    src.write_text('#include "picgpu.hpp"\n#include <cstdio>\nint main() {\n  std::vector<picgpu::StepMetrics> v;\n'
                   + rows + '\n  std::printf("%s", picgpu::report_csv(v).c_str());\n'
                   '  std::printf("%s\\n", picgpu::report_json(v).c_str());\n'
                   '  std::printf("%s\\n", picgpu::report_json({}).c_str());\n}\n')
    exe = tmp_path / "r"
    subprocess.run(["g++", "-std=gnu++20", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    m = _metrics(pg)
    assert out == report_csv(m) + dump_json(report_json(m)) + "\n" + dump_json(report_json([])) + "\n"
