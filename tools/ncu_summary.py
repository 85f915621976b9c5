"""Summarise ncu reports of the streaming kernels into profiles/.

    python tools/ncu_summary.py traffic OUT.json REP1.ncu-rep [REP2 ...]
        per-report (one batch size each) DRAM bytes / duration of every
        captured stream_kernel launch, the algorithmic bytes of the block
        (traffic.cpp:70-76 + 82-94 at 2 B/element) and their ratio; bench.py
        reads `dram_bytes_per_launch` for roofline.traffic.
    python tools/ncu_summary.py launches OUT.md LAUNCHES.csv
        the launch list (ncu --metrics gpu__time_duration.sum) grouped by
        kernel name: count, total µs, share.

Report names must carry the shape: ..._B<b>_dm<dm>_df<df>.ncu-rep (dm/df
default to Llama-3.1-8B).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
]


def raw_rows(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


def to_num(v, unit=""):
    try:
        x = float(str(v).replace(",", ""))
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "us": 1, "ms": 1e3,
             "usecond": 1, "msecond": 1e3, "KB": 1024, "MB": 1024 ** 2}.get(unit, 1)
    return x * scale


def shape_of(rep):
    b = int(re.search(r"_B(\d+)", rep).group(1))
    m = re.search(r"_dm(\d+)", rep)
    n = re.search(r"_df(\d+)", rep)
    return b, int(m.group(1)) if m else 4096, int(n.group(1)) if n else 14336


def traffic(out, reps):
    res = {"source": "ncu --set full --clock-control none (cold L2, serialised launches)",
           "per_batch": {}}
    means = []
    for rep in reps:
        B, dm, df = shape_of(rep)
        alg = 2 * (3 * dm * df + 2 * B * dm + 2 * B * df)
        launches = []
        for d in raw_rows(rep):
            if "stream_kernel" not in d.get("Kernel Name", ""):
                continue
            u = d["_units"]
            e = {k: to_num(d.get(k), u.get(k, "")) for k in METRICS if k in d}
            e["kernel"] = d["Kernel Name"][:80]
            launches.append(e)
        if not launches:
            continue
        rd = sum(x["dram__bytes_read.sum"] for x in launches) / len(launches)
        wr = sum(x["dram__bytes_write.sum"] for x in launches) / len(launches)
        us = sum(x["gpu__time_duration.sum"] for x in launches) / len(launches)
        res["per_batch"][str(B)] = {
            "d_model": dm, "d_ff": df, "launches": len(launches),
            "dram_read_bytes": round(rd), "dram_write_bytes": round(wr),
            "dram_bytes_per_launch": round(rd + wr), "algorithmic_bytes": alg,
            "dram_over_algorithmic": round((rd + wr) / alg, 4),
            "duration_us_cold": round(us, 2),
            "dram_gbs_cold": round((rd + wr) / (us * 1e-6) / 1e9, 1),
            "metrics_first_launch": launches[0],
        }
        means.append(rd + wr)
    res["dram_bytes_per_launch_sweep_mean"] = round(sum(means) / len(means)) if means else None
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: {kk: v[kk] for kk in ("dram_bytes_per_launch", "algorithmic_bytes",
                                                 "dram_over_algorithmic", "duration_us_cold")}
                      for k, v in res["per_batch"].items()}, indent=1))


def launches(out, path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = to_num(r["Metric Value"], r.get("Metric Unit", ""))
        agg[r["Kernel Name"]][0] += 1
        agg[r["Kernel Name"]][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as f:
        f.write("| launches | total µs | share | kernel |\n|---:|---:|---:|---|\n")
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {n} | {us:.1f} | {100 * us / tot:.1f}% | `{k[:90]}` |\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
    else:
        launches(sys.argv[2], sys.argv[3])
