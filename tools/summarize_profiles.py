"""Summarise one measurement campaign (tools/profile_round.sh) into
profiles/<round>/: bench lines, the ncu metrics that the roofline cites
(per kernel), the launch list, and profiles/traffic.json (DRAM bytes per
launch of each dominant kernel, read by bench.py).

    python tools/summarize_profiles.py r01
"""
import csv
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("gpc__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]
# capture name -> (traffic.json key, kernel label used by bench.py)
TRAFFIC = {
    "cfg5_fp4k_gemm": ["cfg5:auto:fp4k gemm", "cfg5:fp4k:fp4k gemm"],
    "cfg3_fp4k_gemm": ["cfg3:auto:fp4k gemm", "cfg3:fp4k:fp4k gemm"],
    "cfg4_fp4k_gemm": ["cfg4:auto:fp4k gemm", "cfg4:fp4k:fp4k gemm"],
    "cfg5_i8_gemm": ["cfg5:i8:i8 gemm"],
    "cfg1_polymul": ["cfg1:auto:polymul_k4"],
    "cfg2_gf_dot": ["cfg2:auto:gf_dot"],
    "redq": ["redq:reduce_words"],
    "pack": ["pack:pack_rows_u8"],
    "unpack": ["unpack:unpack_rows_u8"],
    "polylong": ["polylong:polymul conv"],
}
# measured ceilings / host-path probes written by profile_round.sh, copied verbatim
PROBES = ["copy_floor.jsonl", "pipe_peaks.json", "fp4_library_ceiling.json", "hbm_write_probe.json", "e2e_probe.txt",
          "pageable_probe.txt"]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return int(round(float(v) * scale))


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = os.path.join(ROOT, "gpurun_out", rnd)
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    lines = ["# Measurement summary (%s)" % rnd, "",
             "Produced by `tools/profile_round.sh %s` on one B200 + `tools/summarize_profiles.py %s`." % (rnd, rnd),
             "ncu numbers are single cold-cache launches under the profiler (`--clock-control none`);",
             "bench numbers are CUDA-event timings without the profiler.", "", "## bench lines", "",
             "| file | ms/step | value | dominant kernel | achieved | frac | e2e ms | kernels ms/step |",
             "|---|---|---|---|---|---|---|---|"]
    for f in sorted(glob.glob(os.path.join(src, "bench_*.json"))):
        t = open(f).read().strip()
        if not t:
            continue
        d = json.loads(t.splitlines()[-1])
        shutil.copy(f, dst)
        r = d.get("roofline") or {}
        lines.append("| %s | %.4f | %.4g %s | %s | %s %s | %s | %.2f | %s |" % (
            os.path.basename(f), d["ms_per_step"], d["value"], d["unit"], r.get("kernel"), r.get("achieved"),
            r.get("unit"), r.get("frac"), (d.get("e2e") or {}).get("ms_per_step", float("nan")),
            json.dumps(r.get("kernels_ms_per_step"))))
    lines += ["", "## ncu (one `--set full` capture per kernel)", "",
              "| capture | " + " | ".join(m[1] for m in METRICS) + " |", "|---" * (len(METRICS) + 1) + "|"]
    traffic = {"_doc": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from one "
                       "ncu --set full capture (profiles/%s/*_raw.csv); keys cfg:engine:kernel" % rnd}
    for f in sorted(glob.glob(os.path.join(src, "*_raw.csv"))):
        name = os.path.basename(f)[:-len("_raw.csv")]
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            continue
        h, u, v = rows[0], rows[1], rows[2]
        d, U = dict(zip(h, v)), dict(zip(h, u))
        lines.append("| %s | " % name + " | ".join("%s %s" % (d.get(k, "-"), U.get(k, "")) for k, _ in METRICS) + " |")
        shutil.copy(f, dst)
        det = os.path.join(src, name + "_details.csv")
        if os.path.exists(det):
            shutil.copy(det, dst)
        if name in TRAFFIC and "dram__bytes_read.sum" in d:
            tb = to_bytes(d["dram__bytes_read.sum"], U["dram__bytes_read.sum"]) + \
                to_bytes(d["dram__bytes_write.sum"], U["dram__bytes_write.sum"])
            for key in TRAFFIC[name]:
                traffic[key] = tb
    for f in glob.glob(os.path.join(src, "launches_*.csv")):
        shutil.copy(f, dst)
        lines += ["", "## launch list (`%s`)" % os.path.basename(f), ""]
        txt = open(f).read()
        i = txt.find('"ID"')
        rows = list(csv.reader(txt[i:].splitlines())) if i >= 0 else []
        if rows:
            h = rows[0]
            ki, vi = h.index("Kernel Name"), h.index("Metric Value")
            agg = {}
            for r in rows[1:]:
                if len(r) > vi:
                    nm = r[ki].split("(")[0].split("<")[0].replace("void ", "")
                    c, tot = agg.get(nm, (0, 0.0))
                    agg[nm] = (c + 1, tot + float(r[vi].replace(",", "")))
            tot_all = sum(t for _, t in agg.values())
            lines += ["| kernel | launches | total ns | share |", "|---|---|---|---|"]
            for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
                lines.append("| %s | %d | %.0f | %.3f |" % (nm, c, t, t / tot_all))
    for name in PROBES:
        f = os.path.join(src, name)
        if os.path.exists(f) and os.path.getsize(f):
            shutil.copy(f, dst)
            lines += ["", "## %s" % name, "", "```", open(f).read().strip(), "```"]
    open(os.path.join(dst, "SUMMARY.md"), "w").write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
