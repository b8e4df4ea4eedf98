"""GPU rows in the reference's report schema ("next"
row 2): `BenchReport` (P/include/spten/report.hpp:21-44) with variant "gpu",
emitted in the field order of emit_json / emit_csv (P/src/report.cpp), so GPU
and CPU numbers sit in one table and the flops/gflops columns stay valid."""
from __future__ import annotations

import json
import socket
from typing import List, Optional, Sequence

# P/src/report.cpp emit_json field order
FIELDS = ["tensor", "dims", "nnz", "kernel", "op", "mode", "variant", "strategy", "threads",
          "rank", "runs", "times_s", "mean_s", "sort_s", "preprocess_s", "flops", "gflops",
          "cost", "crosscheck", "host", "precision", "max_threads"]


def bench_report(tensor: str, dims: Sequence[int], nnz: int, kernel: str, times_s: List[float],
                 flops: int, op: Optional[str] = None, mode: Optional[str] = None,
                 strategy: Optional[str] = None, rank: int = 0, sort_s: float = 0.0,
                 preprocess_s: float = 0.0, crosscheck: Optional[str] = None) -> dict:
    mean = sum(times_s) / len(times_s) if times_s else 0.0
    return {
        "tensor": tensor, "dims": [int(d) for d in dims], "nnz": int(nnz), "kernel": kernel,
        "op": op, "mode": mode, "variant": "gpu", "strategy": strategy,
        "threads": 1, "rank": rank or None, "runs": len(times_s), "times_s": list(times_s),
        "mean_s": mean, "sort_s": sort_s, "preprocess_s": preprocess_s, "flops": int(flops),
        "gflops": (flops / mean / 1e9) if mean > 0 else 0.0, "cost": None,
        "crosscheck": crosscheck, "host": socket.gethostname(), "precision": "f32",
        "max_threads": 1,
    }


def emit_json(reports: List[dict]) -> str:
    return json.dumps([{k: r[k] for k in FIELDS} for r in reports], indent=2) + "\n"


# P/src/report.cpp:80-106 emit_csv column order (cost split into 4 columns,
# times_s last).
CSV_COLS = ["tensor", "dims", "nnz", "kernel", "op", "mode", "variant", "strategy", "threads",
            "rank", "runs", "mean_s", "sort_s", "preprocess_s", "flops", "gflops",
            "storage_bytes", "work_flops", "traffic_bytes", "arithmetic_intensity",
            "crosscheck", "host", "precision", "max_threads", "times_s"]


def emit_csv(reports: List[dict]) -> str:
    """Header + one line per report; dims joined with 'x', times_s with ';',
    absent fields empty (P/src/report.cpp emit_csv)."""
    lines = [",".join(CSV_COLS)]
    for r in reports:
        cost = r.get("cost") or {}
        vals = []
        for c in CSV_COLS:
            v = cost.get(c) if c in ("storage_bytes", "work_flops", "traffic_bytes",
                                     "arithmetic_intensity") else r[c]
            if v is None:
                vals.append("")
            elif c == "dims":
                vals.append("x".join(str(d) for d in v))
            elif c == "times_s":
                vals.append(";".join(repr(t) for t in v))
            else:
                vals.append(str(v))
        lines.append(",".join(vals))
    return "\n".join(lines) + "\n"
