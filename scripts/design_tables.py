"""Print DESIGN.md's round-2 measurement table (§4.2) and config-5 sweep table
(§6.1) from the committed bench lines under profiles/ (so the tables can be
regenerated from the evidence)."""
import json
from pathlib import Path

P = Path(__file__).resolve().parents[1] / "profiles"


def line(f):
    return json.loads((P / f).read_text().strip().splitlines()[-1])


def bench_table():
    spec = [("C2 10k x 500, P=4096", "r2_final_bench_c2.json", ""),
            ("**C3 20k x 1000, P=16384** (headline)", "r2_final_bench_c3.json", "b"),
            ("C3, 200 steps", "r2_final_bench_c3_200.json", ""),
            ("C3, index disabled (`--path plane`)", "r2_final_bench_c3_plane.json", ", smem-bound"),
            ("**C4 200k x 2000, P=32768, lazy index (default)**", "r2_final_bench_c4.json", "b"),
            ("C4, full index (budget raised to 120 GB)", "r2_bench_c4_full_index_pipelined.json", ""),
            ("C5 1M x 64, P=1024, L=16", "r2_final_bench_c5.json", ", L2 reuse: every read %.0f GB/s"),
            ("SPEC 20k x 250, P=392", "r2_final_bench_spec.json", ", latency-bound")]
    out = ["| config | kernel | kernel ms | evals/s | row-checks/s | e2e evals/s | physical GB/s (frac) | 200-gen GA e2e evals/s |",
           "|---|---|---|---|---|---|---|---|"]
    for name, f, note in spec:
        d = line(f)
        rf = d["roofline"]
        bold = note == "b"
        if "%" in note:
            note = note % rf["reads_gbs"]
        note = "" if bold else note
        kern = rf["kernel"].split(" (")[0] + (" (lazy)" if "lazy" in rf["kernel"] else "")
        v = ("**%.3g**" if bold else "%.3g") % d["value"]
        fr = ("**%.2f**" if bold else "%.2f") % rf["frac"]
        out.append(f"| {name} | {kern} | {rf['kernel_avg_ms']:.4f} | {v} | {d['row_checks_per_s']:.2g} | "
                   f"{d['e2e']['value']:.3g} | {rf['achieved']:.0f} ({fr}{note}) | {d['amortized']['ga_run']['e2e']:.3g} |")
    return "\n".join(out)


def sweep_table():
    pts = {}
    for ln in (P / "r2_final_sweep_c5.jsonl").read_text().splitlines():
        if ln.startswith("{"):
            d = json.loads(ln)
            pts[(d["rows"], d["L"], d["approx"])] = d
    Ls = sorted({k[1] for k in pts})
    Rs = sorted({k[0] for k in pts})
    out = ["| rows | index | roofline | kernel | " + " | ".join(f"L={L}" for L in Ls) + " |",
           "|---|---|---|---|" + "---|" * len(Ls)]
    for R in Rs:
        d0 = pts[(R, Ls[0], 0.03)]
        kern = sorted({pts[(R, L, 0.03)]["kernel"].replace("table_count_", "").replace("_kernel", "") for L in Ls})
        kern = ["cta" if k == "kernel" else k for k in kern]
        cells = ["%.2f / %.2g" % (pts[(R, L, 0.03)]["frac"], pts[(R, L, 0.03)]["evals_per_s"]) for L in Ls]
        out.append(f"| {R:,} | {d0['index_bytes'] / 1e6:.3g} MB | {d0['regime'].upper()} | {', '.join(kern)} | "
                   + " | ".join(cells) + " |")
    mx = max(abs(pts[(R, L, 0.0)]["evals_per_s"] / pts[(R, L, 0.03)]["evals_per_s"] - 1) for R in Rs for L in Ls)
    return "\n".join(out), mx


if __name__ == "__main__":
    print(bench_table())
    t, mx = sweep_table()
    print()
    print(t)
    print(f"\nmax |approx 0 / approx 0.03 - 1| = {mx:.4f}")
