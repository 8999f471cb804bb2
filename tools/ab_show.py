"""Prints gpurun_out/ab.log (tools/ab.sh) one line per run."""
import json
import sys

lab = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.log"):
    if line.startswith("lib "):
        lab = line.split()[1].split("/")[-1]
        continue
    try:
        d = json.loads(line)
    except ValueError:
        continue
    print(f"{lab:22s} {d['workload']} step {d['graph_step_ms'] * 1e3:7.1f} us",
          {k: round(v * 1e3, 1) for k, v in d["split_ms"].items()})
