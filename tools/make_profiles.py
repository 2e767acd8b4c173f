"""Turn gpurun_out/ ncu captures + the bench line into committed summaries under profiles/.

python tools/make_profiles.py <round-tag> [capture-dir]   (default capture dir: gpurun_out/<round-tag>)
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "smem_dyn_bytes": ("launch__shared_mem_per_block_dynamic", None),
    "sm_clock_hz": ("sm__cycles_elapsed.avg.per_second", None),
    "inst_executed": ("smsp__inst_executed.sum", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "hz": 1, "Khz": 1e3, "Mhz": 1e6,
              "Ghz": 1e9}


TAG = ""


def raw(path):
    exported = path[:-len(".ncu-rep")] + ".raw.csv"  # exported on the box (large reports stay there)
    if os.path.exists(exported):
        out = open(exported).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(path, what):
    h, units, rows = raw(path)
    r = rows[0]
    # the committed copy (profiles/<tag>/ncu/: gzipped raw page, details page, SASS source page)
    d = {"kernel": r[h.index("Kernel Name")], "what": what,
         "report": f"{TAG}/ncu/" + os.path.basename(path)[:-len(".ncu-rep")] + ".raw.csv.gz"}
    for k, (m, scale) in KEYS.items():
        if m not in h:
            continue
        v = float(r[h.index(m)].replace(",", ""))
        u = units[h.index(m)].split("/")[0]
        if scale is None:
            v *= UNIT_SCALE.get(u, 1)
        elif k == "duration_us":
            v = v * {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1)
        d[k] = v
    d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
    return d


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    return tot, cnt


def launch_summary(src, dst):
    tot, cnt = launches(src)
    T = sum(tot.values())
    with open(dst, "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none of `python bench.py --steps 1 "
                 "--warmup 3 --skip-prefill --skip-quant --skip-calib --skip-7b --skip-e2e --skip-cpu "
                 "--skip-gates` (the headline decode step: 48 layers x 4 linears x M in {1,4,16}, plus "
                 "setup/quantize and per-M passes; cold-cache, serialised launches: compare shares, not "
                 "absolutes)\n")
        for k, v in sorted(tot.items(), key=lambda t: -t[1]):
            fh.write(f"{k[:80]:80s} n={cnt[k]:5d} total_us={v / 1e3:10.1f} share={100 * v / T:5.1f}% "
                     f"avg_us={v / cnt[k] / 1e3:8.2f}\n")


def main():
    global TAG
    tag = TAG = sys.argv[1]
    if tag == "launches-only":  # <csv> <out.txt>: summarise an ncu launch list where it was taken
        launch_summary(sys.argv[2], sys.argv[3])
        return
    global OUT
    OUT = sys.argv[2] if len(sys.argv) > 2 else os.path.join(OUT, tag)
    def gemm_b(M, K, N):
        return K * N // 2 + 4 * N * (K // 128) + 2 * M * K + 2 * M * N
    caps = [("decode", "prof_decode_m1_gateup.ncu-rep", "decode GEMM, M=1, K=8192, N=44032 (34B gate|up)",
             gemm_b(1, 8192, 44032)),
            ("decode_m16", "prof_decode_m16_gateup.ncu-rep", "decode GEMM, M=16, K=8192, N=44032",
             gemm_b(16, 8192, 44032)),
            ("decode_m1_oproj", "prof_decode_m1_oproj.ncu-rep", "decode GEMM, M=1, K=8192, N=8192 (34B o_proj)",
             gemm_b(1, 8192, 8192)),
            ("prefill", "prof_prefill_gate.ncu-rep", "prefill GEMM, M=2048, K=8192, N=22016",
             gemm_b(2048, 8192, 22016)),
            ("prefill_m32", "prof_prefill_m32_gateup.ncu-rep", "prefill GEMM, M=32, K=8192, N=44032 (mid-M)",
             gemm_b(32, 8192, 44032)),
            ("decode_m1_qkv", "prof_decode_m1_qkv_r02c.ncu-rep", "decode GEMM, M=1, K=8192, N=10240 (34B qkv)",
             gemm_b(1, 8192, 10240)),
            ("decode_m1_u4", "prof_decode_m1_gateup_u4.ncu-rep",
             "decode GEMM, M=1, K=8192, N=44032, packed u4 zero points (SQ_ZEROS_U4)",
             gemm_b(1, 8192, 44032) - 3 * 44032 * 64 // 2),
            ("quantize", "prof_quant.ncu-rep", "quantize/pack, N=22016, K=8192, with s",
             2 * 22016 * 8192 + 4 * 8192 + 22016 * 8192 // 2 + 4 * 22016 * 64)]
    summ = {"round": tag, "how": "ncu --set full --clock-control none --import-source on (cold cache, "
                                   "one launch after warm-up) via tools/ncu_target.py"}
    for key, f, what, alg in caps:
        p = os.path.join(OUT, f)
        if os.path.exists(p) or os.path.exists(p[:-len(".ncu-rep")] + ".raw.csv"):
            summ[key] = summarise(p, what)
            summ[key]["algorithmic_bytes"] = alg
            summ[key]["traffic_over_algorithmic"] = summ[key]["dram_bytes_per_launch"] / alg
    with open(os.path.join(PROF, f"ncu_summary_{tag}.json"), "w") as fh:
        json.dump(summ, fh, indent=1)
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as fh:
        json.dump(summ, fh, indent=1)
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(os.path.join(OUT, "launches.txt")):  # summarised on the box
        with open(os.path.join(OUT, "launches.txt")) as src, open(os.path.join(PROF, f"launches_{tag}.txt"), "w") as fh:
            fh.write(src.read())
    elif os.path.exists(lp):
        tot, cnt = launches(lp)
        T = sum(tot.values())
        with open(os.path.join(PROF, f"launches_{tag}.txt"), "w") as fh:
            fh.write("ncu --metrics gpu__time_duration.sum --clock-control none of `python bench.py --steps 1 "
                     "--warmup 3 --skip-prefill --skip-quant --skip-calib --skip-7b --skip-e2e --skip-cpu "
                     "--skip-gates` (the headline decode step: 48 layers x 4 linears x M in {1,4,16}, plus "
                     "setup/quantize and per-M passes; cold-cache, serialised launches: compare shares, not "
                     "absolutes)\n")
            for k, v in sorted(tot.items(), key=lambda t: -t[1]):
                fh.write(f"{k[:80]:80s} n={cnt[k]:5d} total_us={v / 1e3:10.1f} share={100 * v / T:5.1f}% "
                         f"avg_us={v / cnt[k] / 1e3:8.2f}\n")
    bp = os.path.join(OUT, "bench.log")
    if os.path.exists(bp):
        lines = [l for l in open(bp) if l.startswith("{")]
        if lines:
            with open(os.path.join(PROF, f"bench_{tag}.json"), "w") as fh:
                fh.write(lines[-1])
    print(json.dumps(summ, indent=1)[:3000])


if __name__ == "__main__":
    main()
