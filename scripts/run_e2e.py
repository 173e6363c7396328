"""End-to-end bicseek::run() -- the UNCHANGED reference evolution engine -- with
the reference CPU evaluator (oracle/_ref/run_ref, WorkerPool of all cores) vs the
B200 evaluator (oracle/_ref/run_device, the drop-in trend TU) vs the
device-aware driver (oracle/_ref/run_device_overlap --engine device; its
archive fed by device-side overlap counts, and -- "lists" -- by host row lists,
EBIC_ARCHIVE_ROWS=1).  Reports run()
wall time (its own steady_clock, evolution.cpp:308,330-331; one tiny warm-up
evaluation before run() keeps CUDA context creation out of it) and checks that
the two produce identical biclusters, generation counts and termination."""
import json
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
CASES = [
    ("config1 default (tabu stop)", []),
    ("config1 forced 200 gens", ["--tabu", "1000000000000"]),
    ("10k x 500, P=4096, 20 gens", ["--rows", "10000", "--cols", "500", "--bic-rows", "500", "--bic-cols", "20",
                                    "--pop", "4096", "--iters", "20", "--tabu", "1000000000000"]),
    ("20k x 1000, P=4096, 10 gens", ["--rows", "20000", "--cols", "1000", "--bic-rows", "500", "--bic-cols", "20",
                                     "--pop", "4096", "--iters", "10", "--tabu", "1000000000000"]),
    ("100k x 2000, P=4096, 5 gens", ["--rows", "100000", "--cols", "2000", "--bic-rows", "2000", "--bic-cols", "20",
                                     "--pop", "4096", "--iters", "5", "--tabu", "1000000000000"]),
]


def run(exe, args, extra=(), trust=True, **env_extra):
    env = dict(os.environ, **env_extra)
    if trust:
        env["EBIC_SHIM_TRUST_POINTER"] = "1"
    else:
        env.pop("EBIC_SHIM_TRUST_POINTER", None)
    out = subprocess.run([str(REPO / "oracle" / "_ref" / exe), "--warm", "1", *extra, *args], check=True, capture_output=True, text=True,
                         env=env, timeout=1800).stdout
    return json.loads(out)


def main():
    print(f"host: {os.cpu_count()} cores")
    for label, args in CASES:
        a, b = run("run_ref", args), run("run_device", args)
        b0 = run("run_device", args, trust=False)  # the default drop-in: cached matrix verified on every call
        c = run("run_device_overlap", args, ("--engine", "device"))
        d = run("run_device_overlap", args, ("--engine", "device"), EBIC_ARCHIVE_ROWS="1")
        same = all(x["result"] == a["result"] and x["generations"] == a["generations"] and
                   x["termination"] == a["termination"] for x in (b, b0, c, d))
        print(f"{label:30s} gens {a['generations']:4d} {a['termination']:9s} CPU ref {a['wall_s']:7.3f} s | "
              f"B200 drop-in TU default env {b0['wall_s']:7.3f} s ({a['wall_s'] / max(b0['wall_s'], 1e-9):5.2f}x) | "
              f"trusted pointer {b['wall_s']:7.3f} s ({a['wall_s'] / max(b['wall_s'], 1e-9):5.2f}x) | "
              f"B200 device driver {c['wall_s']:7.3f} s ({a['wall_s'] / max(c['wall_s'], 1e-9):5.2f}x) | "
              f"lists {d['wall_s']:7.3f} s | "
              f"identical={same}")
        sys.stdout.flush()


if __name__ == "__main__":
    main()
