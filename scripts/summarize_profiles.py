"""Summarise one scripts/gpu_measure.sh pass (gpurun_out/) into profiles/<round>/:
  launches_bench_cfg3.csv   the ncu launch list (gpu__time_duration.sum per launch)
  launch_shares_cfg3.csv    per-kernel totals and shares of the step
  <name>_raw.csv / <name>_details.csv  `ncu -i --page raw|details --csv` of the full captures
  profiles/gs_traffic.json  dram read+write bytes of the GS launch (bench.py's roofline.traffic)
Usage: python scripts/summarize_profiles.py [round_dir=profiles/r01]"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, sys.argv[1] if len(sys.argv) > 1 else "profiles/r01")
RUN = os.path.join(ROOT, "gpurun_out")


def launch_shares():
    src = os.path.join(RUN, "launches.csv")
    rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
    head, body = rows[0], rows[1:]
    ik, iv = head.index("Kernel Name"), head.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in body:
        tot[r[ik]] += float(r[iv].replace(",", "")) / 1e6   # ns -> ms
        cnt[r[ik]] += 1
    all_ms = sum(tot.values())
    with open(os.path.join(OUT, "launch_shares_cfg3.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_ms", "share"])
        for k in sorted(tot, key=lambda k: -tot[k]):
            w.writerow([k.split("(")[0], cnt[k], f"{tot[k]:.3f}", f"{tot[k] / all_ms:.4f}"])
    with open(os.path.join(OUT, "launches_bench_cfg3.csv"), "w") as f:
        f.write(open(src).read())


def export(rep, name):
    path = os.path.join(RUN, rep)
    if not os.path.exists(path):
        return None
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(os.path.join(OUT, f"{name}_raw.csv"), "w").write(raw)
    open(os.path.join(OUT, f"{name}_details.csv"), "w").write(det)
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    # several captured launches (the residual GS runs one launch per size class of a band):
    # times and bytes summed, rates from the first
    vals = rows[2:]
    v = list(vals[0])
    for key in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
        if key in h and len(vals) > 1:
            i = h.index(key)
            v[i] = str(sum(float(r[i].replace(",", "")) for r in vals if len(r) > i))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
             "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12}

    def get(k):   # bytes, or milliseconds for times
        if k not in h:
            return None
        i = h.index(k)
        return float(v[i].replace(",", "")) * scale.get(u[i], 1.0)
    return {"ms": get("gpu__time_duration.sum"),
            "dram_read": get("dram__bytes_read.sum"), "dram_write": get("dram__bytes_write.sum"),
            "tensor_pct": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "l2_hit": get("lts__t_sector_hit_rate.pct")}


def main():
    os.makedirs(OUT, exist_ok=True)
    launch_shares()
    summary = {}
    for rep, name in (("gs_full.ncu-rep", "rgs_full"), ("psf_full.ncu-rep", "psf_tc_full"),
                      ("das_full.ncu-rep", "das_full")):
        summary[name] = export(rep, name)
    print(json.dumps(summary, indent=1))
    gs = summary.get("rgs_full")
    if gs and gs["dram_read"] is not None:
        # the default bench variant (bench.variant_key) on the residual kernel (gs_kernel 4)
        tp = os.path.join(ROOT, "profiles", "gs_traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        rel = os.path.relpath(os.path.join(OUT, "rgs_full_raw.csv"), ROOT)
        d["cfg3|order1|dr0|alt0|csm|n1|g1"] = {
            "dram_bytes": gs["dram_read"] + gs["dram_write"], "gs_kernel": 4,
            "source": f"{rel} (rgs_kernel, the band's launches summed: dram read {gs['dram_read'] / 1e6:.1f} MB + write "
                      f"{gs['dram_write'] / 1e6:.1f} MB, L2 hit {gs['l2_hit']:.1f} %)"}
        json.dump(d, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
