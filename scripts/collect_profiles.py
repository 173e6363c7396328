"""Copy one round's GPU-check outputs (gpurun_out/*_<tag>*) into profiles/:
bench lines, ncu summaries, launch-list summary, run() e2e, test / smoke logs,
and refresh profiles/ncu_traffic.json from the raw ncu exports.
usage: python scripts/collect_profiles.py TAG"""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
OUT, PROF = REPO / "gpurun_out", REPO / "profiles"
tag = sys.argv[1]
for f in OUT.glob(f"bench*_{tag}.json"):
    name = f.name.replace(f"_{tag}.json", "").replace("bench_", "").replace("bench", "c3")
    shutil.copy(f, PROF / f"{tag}_bench_{name}.json")
for src, dst in ((f"run_e2e_{tag}.txt", f"{tag}_run_e2e.txt"), (f"pytest_gpu_{tag}.log", f"{tag}_pytest_gpu.log"),
                 (f"smoke_{tag}.log", f"{tag}_smoke.log"), (f"gpu_{tag}.txt", f"{tag}_gpu.txt")):
    if (OUT / src).exists():
        shutil.copy(OUT / src, PROF / dst)
traffic = json.loads((PROF / "ncu_traffic.json").read_text()) if (PROF / "ncu_traffic.json").exists() else {}
for f in sorted(OUT.glob(f"prof_*_{tag}.raw.csv")):
    cfg = f.name[len("prof_"):-len(f"_{tag}.raw.csv")]
    summ = subprocess.run([sys.executable, str(REPO / "scripts" / "ncu_summ.py"), str(f)], capture_output=True,
                          text=True).stdout
    (PROF / f"{tag}_ncu_{cfg}.txt").write_text(
        f"# ncu --set full --clock-control none (1 launch, cold cache), round {tag}\n" + summ)
    if cfg in ("c2", "c3", "c4", "c5"):
        rows = list(csv.reader(f.open()))
        h, u, v = rows[0], rows[1], rows[2]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def val(k):
            return float(v[h.index(k)].replace(",", "")) * scale.get(u[h.index(k)], 1)

        t = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
        t *= {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(
            u[h.index("gpu__time_duration.sum")], 1)
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        traffic[cfg] = {"kernel": v[h.index("Kernel Name")][:70], "dram_bytes_per_launch": rd + wr,
                        "dram_read_bytes": rd, "dram_write_bytes": wr, "ncu_duration_s": t,
                        "source": f"profiles/{tag}_ncu_{cfg}.txt (ncu --set full --clock-control none, 1 launch)"}
(PROF / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1))
launches = OUT / f"launches_c3_{tag}.csv"
if launches.exists():
    s = subprocess.run([sys.executable, str(REPO / "scripts" / "launch_summ.py"), str(launches)], capture_output=True,
                       text=True).stdout
    (PROF / f"{tag}_launches_c3_summary.txt").write_text(
        "# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 3 --warmup 3 "
        "--no-cpu-baseline (c3)\n# cold-cache, serialised launches: compare SHARES, not absolutes\n" + s)
print("collected", tag)
