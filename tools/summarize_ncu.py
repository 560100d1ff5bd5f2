"""Summarise ncu CSV exports (from gpurun_out/) into profiles/ (tracked).

  python tools/summarize_ncu.py launches <launches.csv> <out.md>
  python tools/summarize_ncu.py kernel <raw.csv> <details.csv> <label> <out.json>
"""
import collections
import csv
import json
import sys


def _open(path):
    if path.endswith(".gz"):
        import gzip
        return gzip.open(path, "rt")
    return open(path)


def _table(path):
    rows = list(csv.reader(_open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r or "ID" in r[:1]:
            return rows[i], rows[i + 1:]
    return rows[0], rows[1:]


def launches(path, out):
    h, rows = _table(path)
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "nsecond": 1e-3, "usecond": 1.0,
              "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | total (us) | share | avg (us) |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {t / tot:.3f} | {t / c:.1f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "fp64_pipe_pct_active": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_inst_pct_active": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "registers_per_thread": "launch__registers_per_thread",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_slots_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "sm_mhz": "smsp__cycles_elapsed.avg.per_second",
    "inst_executed": "smsp__inst_executed.sum",
    "local_load_requests": "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum",
}
STALLS = ["no_instruction", "wait", "not_selected", "math_pipe_throttle", "long_scoreboard",
          "short_scoreboard", "branch_resolving", "dispatch_stall", "barrier", "mio_throttle",
          "lg_throttle", "tex_throttle", "drain", "membar", "sleeping", "misc"]


def kernel(raw, details, label, out):
    rows = list(csv.reader(open(raw)))
    h, units, vals = rows[0], rows[1], rows[2]
    get = {n: (vals[i], units[i]) for i, n in enumerate(h)}
    res = {"label": label, "kernel": get.get("Kernel Name", ("?",))[0],
           "grid": get.get("Grid Size", ("?",))[0], "block": get.get("Block Size", ("?",))[0]}

    def num(name):
        v, u = get.get(name, (None, None))
        if v is None:
            return None
        try:
            f = float(v.replace(",", ""))
        except ValueError:
            return None
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "Kbyte": 1e3, "Mbyte": 1e6,
                 "Gbyte": 1e9, "byte": 1.0, "Ghz": 1e3, "Mhz": 1.0}
        return f * scale.get(u, 1.0)

    for k, name in KEYS.items():
        res[k] = num(name)
    res["dram_bytes_per_launch"] = ((res["dram_read_bytes"] or 0) + (res["dram_write_bytes"] or 0)
                                    if res.get("dram_read_bytes") is not None else None)
    res["stalls_per_issue"] = {}
    for s in STALLS:
        v = num(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
        if v is not None and v >= 0.01:
            res["stalls_per_issue"][s] = round(v, 3)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kernel(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5])
