"""Summarise an ncu launch list + one `--set full` capture into profiles/.

usage: python tools/ncu_summarize.py <launches.csv> <capture.ncu-rep> <key> [<out_dir>]

* launch shares: median device time per libmhb step kernel (plan_*, sign_kernel,
  finalize_kernel) over the captured launches, as a share of their sum (ncu times are
  cold-cache and serialised: compare shares, not absolutes);
* the capture's DRAM bytes, pipe utilisation, occupancy and stall ratios.
Writes profiles/ncu_summary.json[<key>] (read by bench.py for roofline.traffic) and
<out_dir>/ncu_<kernel>_<key>.txt (ncu --page details).
"""
import csv
import io
import json
import re
import statistics
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

STEP = ("plan_count", "plan_scan", "plan_scatter", "plan_small", "sign_kernel", "sign_gap_kernel", "finalize_kernel")


def _is_step(name):
    """The timed step's kernels: the plan, the signature kernel (not a BANDS instance:
    bench.py times the fused band-key pass beside the step) and finalize."""
    import re as _re
    if not any(s in name for s in STEP):
        return False
    m = _re.search(r"sign_kernel<(\d+), (\d), (\d), [^,]+, (\d)", name)
    return not (m and m.group(4) == "1")
METRICS = (
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
    "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.per_cycle_active", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
)
PATTERNS = (r"pipe_alu.*pct_of_peak", r"pipe_fma.*pct_of_peak", r"warps_issue_stalled_.*_per_issue_active\.ratio")


def read_launch_csv(path):
    text = Path(path).read_text().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    dur = defaultdict(list)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if not _is_step(name):
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        dur[name].append(v)
    med = {k: statistics.median(v) for k, v in dur.items()}
    tot = sum(med.values())
    return {k: round(v / tot, 4) for k, v in med.items()}, {k: round(v, 4) for k, v in med.items()}


def read_capture(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in raw.splitlines() if l.startswith('"')]
    hdr, units, data = next(csv.reader([lines[0]])), next(csv.reader([lines[1]])), next(csv.reader([lines[2]]))
    out = {}
    for h, u, v in zip(hdr, units, data):
        if any(h.endswith(m) or h == m for m in METRICS) or any(re.search(p, h) for p in PATTERNS):
            out[h] = f"{v} {u}".strip()
    kernel = data[hdr.index("Kernel Name")]
    return kernel, out


def main():
    launches, rep, key = sys.argv[1:4]
    out_dir = Path(sys.argv[4] if len(sys.argv) > 4 else "profiles/r01")
    shares, med_ms = read_launch_csv(launches)
    kernel, m = read_capture(rep)

    def val(name):
        k = next(k for k in m if k.endswith(name))
        return float(m[k].split()[0].replace(",", ""))

    def scaled(name):  # to bytes
        k = next(k for k in m if k.endswith(name))
        v, unit = m[k].split()[0], m[k].split()[-1]
        return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)

    summary_path = Path("profiles/ncu_summary.json")
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    traffic = scaled("dram__bytes_read.sum") + scaled("dram__bytes_write.sum")
    entry = summary.get(key, {})
    entry.update({"kernel": kernel, "dram_bytes_per_launch": traffic,
                  "source": f"{out_dir}/ncu_sign_kernel_{key.split('/')[0]}.txt (ncu --set full, 1 launch)",
                  "launch_share_of_step_ncu": shares, "launch_median_ms_ncu": med_ms, "metrics": m})
    summary[key] = entry
    summary_path.write_text(json.dumps(summary, indent=1) + "\n")
    details = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    (out_dir / f"ncu_sign_kernel_{key.split('/')[0]}.txt").write_text(details)
    print(json.dumps({"kernel": kernel, "traffic": traffic, "shares": shares}, indent=1))


if __name__ == "__main__":
    main()
