"""Summarise ncu outputs into profiles/ (run here, on the CPU side, after a gpurun).

  python tools/ncu_summarize.py --full gpurun_out/prof_top.ncu-rep --key topk \
      --launches gpurun_out/launches.csv --tag r01

Writes profiles/ncu_summary.json (per-kernel DRAM bytes per launch from the
`--set full` capture; bench.py reads the "topk" entry into roofline.traffic),
profiles/<tag>_ncu_<key>.md (headline metrics + stall reasons) and
profiles/<tag>_launches_n1.csv (the launch list: per-launch gpu__time_duration).
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "smsp__inst_executed.sum"]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", required=True)
    ap.add_argument("--key", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--match", default="", help="only launches whose kernel name contains this")
    a = ap.parse_args()
    recs = [(d, u) for d, u in raw(a.full) if a.match in d.get("Kernel Name", "")]
    dram, t = [], []
    lines = [f"# ncu --set full: {a.key} ({os.path.basename(a.full)}, {len(recs)} launch(es) captured)", ""]
    for d, u in recs:
        rd = float(d["dram__bytes_read.sum"]) * UNIT.get(u["dram__bytes_read.sum"], 1.0)
        wr = float(d["dram__bytes_write.sum"]) * UNIT.get(u["dram__bytes_write.sum"], 1.0)
        dram.append((rd, wr))
        t.append(float(d["gpu__time_duration.sum"]))
        lines.append(f"## {d['Kernel Name'][:100]}")
        for k in KEEP:
            if k in d:
                lines.append(f"* {k}: {d[k]} {u.get(k, '')}")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
              for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v.replace(",", "").replace(".", "").isdigit()}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        lines.append("* stall samples: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
        lines.append("")
    n = len(dram)
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ.setdefault("kernels", {})
    summ["kernels"] = {k: v for k, v in summ["kernels"].items()
                       if k in (a.key,) or not (k.startswith("topk_") and k not in ("topk_bucketed",))}
    summ["kernels"][a.key] = {
        "dram_bytes_per_launch": sum(r + w for r, w in dram) / n,
        "dram_read_MB": sum(r for r, _ in dram) / n / 1e6,
        "dram_write_MB": sum(w for _, w in dram) / n / 1e6,
        "time_us": sum(t) / n,
        "launches_captured": n,
        "source": f"{os.path.basename(a.full)} ({a.tag}, ncu --set full --clock-control none, cold caches)",
    }
    json.dump(summ, open(summ_path, "w"), indent=1)
    open(os.path.join(PROF, f"{a.tag}_ncu_{a.key}.md"), "w").write("\n".join(lines))
    if a.launches:
        dst = os.path.join(PROF, f"{a.tag}_launches_n1.csv")
        with open(a.launches) as f:
            body = [l for l in f if l.startswith('"')]
        open(dst, "w").writelines(body)
        # per-kernel share of the launch list
        agg = collections.Counter()
        for r in csv.DictReader(io.StringIO("".join(body))):
            if r.get("Metric Name") == "gpu__time_duration.sum":
                agg[r["Kernel Name"].split("(")[0][:60]] += float(r["Metric Value"])
        ours = {k: v for k, v in agg.items() if "sparcml::" in k}
        tot = sum(ours.values()) or 1.0
        with open(os.path.join(PROF, f"{a.tag}_launches_n1_share.md"), "w") as f:
            f.write(f"# launch list share ({os.path.basename(a.launches)}; ncu per-launch gpu__time_duration, "
                    "cold caches, serialised)\n\nShare of the step's library kernels (the hot path):\n\n")
            for k, v in sorted(ours.items(), key=lambda x: -x[1]):
                f.write(f"* {k}: {v / 1e3:.1f} us total, {100 * v / tot:.1f}%\n")
            f.write("\nHarness kernels in the same run (L2 flush write/read, pre-step spin; outside the timed events):\n\n")
            for k, v in sorted(agg.items(), key=lambda x: -x[1]):
                if k not in ours:
                    f.write(f"* {k}: {v / 1e3:.1f} us total\n")
    print(json.dumps(summ["kernels"][a.key], indent=1))


if __name__ == "__main__":
    main()
