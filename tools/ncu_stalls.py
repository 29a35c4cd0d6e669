"""Summarise an ncu report: per kernel launch, duration, IPC and the
dominant issue-stall reasons (pc sampling)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
          for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
          and v.replace(".", "", 1).isdigit()}
    tot = sum(st.values()) or 1
    top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
    print(d.get("Kernel Name", "")[:28], "dur_ns", d.get("gpu__time_duration.sum"),
          "ipc", d.get("sm__inst_executed.avg.per_cycle_active"),
          " ".join(f"{k}={v / tot:.0%}" for k, v in top))
