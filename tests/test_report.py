"""Reference-schema reporting (paper_1902_03317_b200/report.py) mirrors the
field order of P/src/report.cpp emit_json / emit_csv."""
import json
import os
import re

import pytest

from paper_1902_03317_b200 import report

REPORT_CPP = "/root/reference/proj/src/report.cpp"


def _row():
    return report.bench_report("c2", [10, 20, 30], 1000, "tew_eq", [0.001, 0.002], 1000,
                               op="add")


def test_json_fields_and_values():
    out = json.loads(report.emit_json([_row()]))
    assert list(out[0].keys()) == report.FIELDS
    assert out[0]["variant"] == "gpu" and out[0]["mean_s"] == pytest.approx(0.0015)
    assert out[0]["gflops"] == pytest.approx(1000 / 0.0015 / 1e9)


def test_csv_layout():
    lines = report.emit_csv([_row()]).splitlines()
    assert lines[0].split(",") == report.CSV_COLS
    cells = lines[1].split(",")
    assert cells[1] == "10x20x30" and cells[-1] == "0.001;0.002"


@pytest.mark.skipif(not os.path.exists(REPORT_CPP), reason="reference sources absent")
def test_field_order_matches_reference_source():
    src = open(REPORT_CPP).read()
    json_keys = list(dict.fromkeys(re.findall(r'j\["(\w+)"\]\s*=', src)))  # cost appears twice
    assert json_keys == report.FIELDS
    start = src.index('"tensor,dims')
    stmt = src[start:src.index(";", start)]
    cols = "".join(re.findall(r'"([^"]*)"', stmt)).replace("\\n", "").split(",")
    assert cols == report.CSV_COLS
