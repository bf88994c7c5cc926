"""Copy one tools/final_evidence.sh capture (gpurun_out/ev) into profiles/ under a tag, summarise
the ncu reports and refresh profiles/roofline_traffic.json from the complex128/complex64 K1 captures.
usage: python tools/collect_evidence.py <tag>   (e.g. r02_end)"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EV = os.path.join(ROOT, "gpurun_out", "ev")
PR = os.path.join(ROOT, "profiles")
tag = sys.argv[1]


def cp(src, dst):
    if os.path.exists(os.path.join(EV, src)):
        shutil.copy(os.path.join(EV, src), os.path.join(PR, f"{tag}_{dst}"))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units, v = r[0], r[1], r[2]

    def get(k):
        x = float(v[h.index(k)].replace(",", ""))
        u = units[h.index(k)].lower()
        scale = {"gbyte": 1e9, "mbyte": 1e6, "kbyte": 1e3, "byte": 1.0, "us": 1.0, "ns": 1e-3, "ms": 1e3}.get(u, 1.0)
        return x * scale
    return v[h.index("Kernel Name")], get


for f, d in [("bench.json", "bench.json"), ("bench_ref.json", "bench_reference.json"), ("gputest.log", "gputest.log"),
             ("smoke.log", "smoke.log"), ("launches_bench.csv", "launches_bench.csv"),
             ("km1_c128.ncu-rep", "km1_c2.ncu-rep"), ("krylov_ab.log", "krylov_ab.log"),
             ("k1_timeline_c128.json", "k1_timeline_c128.json"), ("k1_timeline_c64.json", "k1_timeline_c64.json"),
             ("k1_timeline_c128.log", "k1_timeline_c128.log"), ("k1_timeline_c64.log", "k1_timeline_c64.log"),
             ("k1_rdup_ab.log", "k1_rdup_ab.log"), ("krylov_c1.csv", "krylov_c1.csv"), ("krylov_c3.csv", "krylov_c3.csv"),
             ("bcr_c3.csv", "launches_bcr_c3.csv")]:
    cp(f, d)
tr_path = os.path.join(PR, "roofline_traffic.json")
tr = json.load(open(tr_path))
for rep, key, out in [("km1_c128.ncu-rep", "kkt_apply_c128_c2", "ncu_km1_c2.txt"),
                      ("km1_c64.ncu-rep", "kkt_apply_c64_c2", "ncu_km1_c64.txt")]:
    path = os.path.join(EV, rep)
    if not os.path.exists(path):
        continue
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), path],
                         capture_output=True, text=True).stdout
    open(os.path.join(PR, f"{tag}_{out}"), "w").write(
        f"# ncu --set full --clock-control none, tools/prof_kkt.py ({rep}), capture tagged {tag}\n" + txt)
    name, get = raw(path)
    rd, wr, us = get("dram__bytes_read.sum"), get("dram__bytes_write.sum"), get("gpu__time_duration.sum")
    tr[key].update({"dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                    "source": f"profiles/{tag}_{out} (ncu --set full --clock-control none, tools/prof_kkt.py, "
                              f"{us:.1f} us)"})
    print(key, name[:70], f"{us:.1f} us, read {rd / 1e6:.1f} MB, write {wr / 1e6:.1f} MB")
json.dump(tr, open(tr_path, "w"), indent=1)
b = json.load(open(os.path.join(EV, "bench.json")))
k = b["krylov"]
print("bench:", round(b["value"]), "applies/s", round(b["ms_per_step"] * 1e3, 1), "us frac", round(b["roofline"]["frac"], 3),
      "peak", b["roofline"]["peak"], "| c64", round(b["c64"]["ms_per_apply"] * 1e3, 1), "us frac", round(b["c64"]["frac"], 3),
      "| krylov", {n: round(v["iters_per_s"]) for n, v in k.items()}, "| e2e", round(b["e2e"]["value"], 1))
r = json.load(open(os.path.join(EV, "bench_ref.json")))
print("reference arm:", round(r["value"], 1), r["unit"], r["cpu_baseline"]["cores"], "threads")
