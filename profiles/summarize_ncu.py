"""Summarize ncu captures into the committed profile artifacts of a round.

    python profiles/summarize_ncu.py ROUND_DIR LAUNCH_CSV FULL_REP [WORKLOAD] [STEPS]

LAUNCH_CSV  `ncu --metrics gpu__time_duration.sum --clock-control none --csv` of
            `bench.py --steps 1 --warmup 1 --e2e-steps 1` (STEPS decompositions: warmup,
            timed, profiled, e2e warmup, e2e timed = 5).
FULL_REP    `ncu --set full --import-source on --clock-control none -k regex:"k_umma|k_block_sumsq"` of the
            same command.
Writes ROUND_DIR/launches_<workload>_summary.csv (per-kernel share of one step),
ROUND_DIR/ncu_full_<workload>.md (per-launch metrics of the UMMA kernels) and merges
DRAM bytes per launch into ROUND_DIR/ncu_traffic.json (read by bench.py's roofline).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

TAG_OF = {  # k_umma<A_MN, EPI, NT, X3, H> → bench/ProfScope kernel class
    ("0", "1"): "umma_atx_rowsq", ("0", "0"): "umma_atx_store", ("1", "0"): "umma_ax",
}


def tag_of(name):
    if "k_umma2_rowsq" in name:
        return "umma_atx_rowsq"
    if "k_block_sumsq" in name:
        return "block_sumsq"
    if "k_chol_persistent" in name:
        return "chol_inv"
    if "k_jacobi_packed" in name:
        return "sym_eig"
    if "k_copy_segments" in name:
        return "copy_segments"
    for k in ("k_umma2_h3m<", "k_umma2_h3<"):  # CTA-pair 3×FP16 products: <A_MN, EPI>
        if k in name:
            a = name.split(k)[1].split(">")[0].replace("(bool)", "").split(",")[0].strip()
            return "umma_ax_h3" if a in ("1", "true") else "umma_atx_h3"
    if "k_umma<" not in name:
        return None
    args = name.split("k_umma<")[1].split(">")[0].replace("(bool)", "").replace("(int)", "").split(",")
    args = [a.strip().replace("false", "0").replace("true", "1") for a in args]
    if len(args) >= 5 and args[3] == "1" and args[4] == "1":  # 3×FP16 products
        return "umma_ax_h3" if args[0] == "1" else "umma_atx_h3"
    return TAG_OF.get((args[0], args[1]))


def short(name):
    n = name.split("(")[0].replace("void ", "")
    for pre in ("bcur_b200::<unnamed>::", "bcur_b200::(anonymous namespace)::", "bcur_b200::ops::", "unnamed>::"):
        n = n.replace(pre, "")
    return n[:90]


def launches(path, steps):
    if path.endswith(".gz"):
        import gzip
        rows = list(csv.reader(gzip.open(path, "rt")))
    else:
        rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-6)
        tot[short(d["Kernel Name"])] += v
        cnt[short(d["Kernel Name"])] += 1
    return {k: (tot[k] / steps, cnt[k] / steps) for k in tot}


def full(path):
    if path.endswith(".csv.gz"):  # an exported `ncu -i … --page raw --csv`
        import gzip
        out = gzip.open(path, "rt").read()
    elif path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
            "launch__block_size", "launch__registers_per_thread"]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        rec = {"kernel": short(d["Kernel Name"]), "tag": tag_of(d["Kernel Name"])}
        for w in want:
            if w in h:
                u = units[h.index(w)]
                v = float(d[w].replace(",", "")) if d[w] else float("nan")
                if u in ("Kbyte", "KB"):
                    v *= 1e3
                elif u in ("Mbyte", "MB"):
                    v *= 1e6
                elif u in ("Gbyte", "GB"):
                    v *= 1e9
                elif u == "usecond":
                    v *= 1e-3
                elif u == "nsecond":
                    v *= 1e-6
                rec[w] = v
        res.append(rec)
    return res


def main():
    rd, lcsv, rep = sys.argv[1:4]
    workload = sys.argv[4] if len(sys.argv) > 4 else "c3"
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
    L = launches(lcsv, steps)
    total = sum(v[0] for v in L.values())
    with open(os.path.join(rd, f"launches_{workload}_summary.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "ms_per_step", "launches_per_step", "share_of_step"])
        for k, (ms, n) in sorted(L.items(), key=lambda kv: -kv[1][0]):
            w.writerow([k, f"{ms:.4f}", f"{n:g}", f"{ms / total:.4f}"])
    F = full(rep)
    md = [f"# ncu --set full, tensor-core and streaming kernels of one `{workload}` bench step (cold-cache, serialised replay)", "",
          "| kernel | class | ms | DRAM read MB | DRAM write MB | DRAM % | L2 % | tensor % | FMA % | XU % | grid | regs |",
          "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    per_tag = collections.defaultdict(list)
    for r in F:
        md.append("| {kernel} | {tag} | {t:.3f} | {rd:.1f} | {wr:.1f} | {dr:.1f} | {l2:.1f} | {tc:.1f} | {fma:.1f} | {xu:.1f} "
                  "| {g:.0f} | {rg:.0f} |".format(
                      kernel=r["kernel"], tag=r["tag"], t=r.get("gpu__time_duration.sum", 0),
                      rd=r.get("dram__bytes_read.sum", 0) / 1e6, wr=r.get("dram__bytes_write.sum", 0) / 1e6,
                      dr=r.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0),
                      l2=r.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", 0),
                      tc=r.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0),
                      fma=r.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 0),
                      xu=r.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 0),
                      g=r.get("launch__grid_size", 0), rg=r.get("launch__registers_per_thread", 0)))
        if r["tag"]:
            per_tag[r["tag"]].append(r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0))
    with open(os.path.join(rd, f"ncu_full_{workload}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    tp = os.path.join(rd, "ncu_traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    traffic[workload] = {t: sum(v) / len(v) for t, v in per_tag.items()}
    with open(tp, "w") as f:
        json.dump(traffic, f, indent=1)
    print(open(os.path.join(rd, f"launches_{workload}_summary.csv")).read()[:2500])
    print("\n".join(md))


if __name__ == "__main__":
    main()
