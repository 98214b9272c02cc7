"""Turn tools/full_profile.sh outputs (gpurun_out/) into the committed
profile summaries:

  profiles/<tag>_launches.md   ncu launch list of the bench command, per kernel
  profiles/<tag>_ncu.md        key `ncu --set full` metrics of the top kernels
  profiles/ncu_traffic.json    DRAM bytes per launch (bench.py's roofline.traffic)

Usage: python tools/summarize_profiles.py <tag>   (e.g. r1_latest)
"""
import csv
import collections
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x"]


def launches(tag):
    path = os.path.join(OUT, "launches_full.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ii = hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
              "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        per[r[ii]][r[im]] = v
        names[r[ii]] = r[ik]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        k = names[i].split("(")[0][:70]
        a = agg[k]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list — `bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-approx --no-decode` "
             f"(128K, 32 layers; first 700 launches) ({tag})", "",
             "Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none -c 400 --csv` (cold-cache, serialised: compare shares, not absolutes).", "",
             "| kernel | launches | total µs | share | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {a[0]} | {a[1]:.1f} | {a[1] / total:.3f} | {a[2] / 1e6:.1f} | {a[3] / 1e6:.1f} |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")


def raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        out.append(d)
    return out


def ncu_summary(tag):
    lines = [f"# ncu --set full summaries ({tag})", "",
             "Captured with `tools/full_profile.sh` (one 128K prefill layer: `tools/profile_one.py 131072`; one "
             "batched-decode layer step: `tools/decode_probe.py 8 131072 1`; K1: `tools/compress_time.py 131072`, "
             "first launch = the 128K append + compress, second = a re-sync pass).  ncu-serialised (cold L2): compare "
             "against the bench only as shares.", ""]
    traffic = {"source": f"profiles/{tag}_ncu.md: ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per "
                         "launch (tools/full_profile.sh)"}
    for rep, label in (("prefill128k.ncu-rep", "prefill128k"), ("decode_cluster.ncu-rep", "decode"),
                       ("compress.ncu-rep", "k1")):
        path = os.path.join(OUT, rep)
        if not os.path.exists(path):
            continue
        for d in raw(path):
            name = d.get("Kernel Name", ("?", ""))[0]
            lines += [f"## {label}: {name[:90]}", "", "| metric | value | unit |", "|---|---|---|"]
            for k in KEYS:
                if k in d:
                    lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
            lines.append("")

            def nbytes(k):
                v, u = d[k]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                return float(v.replace(",", "")) * scale
            tot = int(nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"))
            if "select_tc" in name:
                traffic["select_tc_kernel (stage-1)"] = {"bytes_per_launch": tot, "launch": "one 131072-row layer"}
            elif "attend_tc" in name or "attend_share" in name:
                traffic["attend (stage-2)"] = {"bytes_per_launch": tot, "launch": "one 131072-row layer (rows >= 2048 "
                                               "on attend_share_kernel)" if "attend_share" in name else
                                               "one 131072-row layer"}
            elif "stream_compress" in name and "stream_compress_kernel" not in traffic:
                traffic["stream_compress_kernel"] = {"bytes_per_launch": tot,
                                                     "launch": "128K-row prefill append + fine/coarse means"}
            elif "decode_cluster" in name:
                traffic["decode_cluster_kernel"] = {"bytes_per_launch": tot,
                                                    "launch": "one layer step, 8 sequences x 128K"}
    open(os.path.join(PROF, f"{tag}_ncu.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "latest"
    launches(tag)
    ncu_summary(tag)
    print("wrote", tag)
