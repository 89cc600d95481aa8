"""Per-stage DRAM traffic and kernel time of one warm Si64 build from an ncu
launch list with NVTX stage names (run under ncu as below, then summarise):

  ncu --nvtx --print-nvtx-rename kernel --profile-from-start off --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --log-file gpurun_out/traffic.csv python tools/prof_build.py
  python tools/stage_traffic.py gpurun_out/traffic.csv profiles/traffic_r01.json

Writes {stage: dram bytes per build} (+ a _detail block) for bench.py's roofline."""
import collections
import csv
import json
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    count = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        stage = r[ki].split("/")[0].strip() if "/" in r[ki] else "(none)"
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        agg[stage][r[mi]] += v
        if r[mi] == "gpu__time_duration.sum":
            count[stage] += 1
    out, detail = {}, {}
    for st, m in agg.items():
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        out[st] = b
        detail[st] = {"dram_read_bytes": m.get("dram__bytes_read.sum", 0.0),
                      "dram_write_bytes": m.get("dram__bytes_write.sum", 0.0),
                      "kernel_ms_serialised": m.get("gpu__time_duration.sum", 0.0) / 1e6, "launches": count[st]}
    out["_detail"] = detail
    out["_note"] = ("ncu launch list of one warm build (tools/prof_build.py), per NVTX stage; per-launch times are "
                    "cold-cache and serialised, so only the stage shares compare with bench.py")
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    for st, d in sorted(detail.items(), key=lambda x: -x[1]["kernel_ms_serialised"]):
        print(f"{st:12s} launches={d['launches']:4d} ms={d['kernel_ms_serialised']:8.3f} "
              f"dram={(d['dram_read_bytes'] + d['dram_write_bytes']) / 1e9:8.3f} GB")


if __name__ == "__main__":
    main()
