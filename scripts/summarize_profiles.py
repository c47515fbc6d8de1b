"""Summarize a round's ncu captures (scripts/profile.sh) into profiles/<tag>/.

  launches_<tag>.csv  ->  per-kernel time / DRAM bytes of one timed GCN step
                          and the kernel shares of the step
  full_<tag>.ncu-rep  ->  key --set full metrics of the captured kernels
Writes profiles/<tag>/summary.md, step_launches.csv, full_metrics.csv and
profiles/traffic.json (DRAM bytes per launch of each captured kernel, read by
bench.py for the roofline `traffic` field).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
SRC = os.path.join(ROOT, "gpurun_out")
DST = os.path.join(ROOT, "profiles", TAG)
os.makedirs(DST, exist_ok=True)


def short(name):
    name = name.replace("void ", "")
    return name.split("(")[0][:70]


def launches(name=None):
    rows = list(csv.reader(open(os.path.join(SRC, name or f"launches_{TAG}.csv"))))
    hdr, data, order = None, {}, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"])
            if key not in data:
                data[key] = {}
                order.append(key)
            data[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [(k[1], data[k]) for k in order]


def one_step(ls):
    """Timed GCN step: k_spmm_lean (A'X) ... k_spmm_lean (A'^T G2).  Take the
    last complete step before the component micro-timings start."""
    idx = [i for i, (n, _) in enumerate(ls) if "k_spmm_lean" in n]
    steps = []
    for a, b in zip(idx[::2], idx[1::2]):
        seg = ls[a:b + 1]
        if any("k_gemm_tc" in n for n, _ in seg):
            steps.append(seg)
    return steps[5] if len(steps) > 5 else steps[-1]


def gat_step(ls):
    """One GAT layer step of scripts/kbench.py gat: X.Theta GEMM (+ split),
    node scores, ... up to the next step's GEMM.  Take the last complete one."""
    # the node scores live in the X.Theta epilogue: a step starts two launches
    # (Theta split + GEMM) before its first attention kernel
    idx = [i for i, (n, _) in enumerate(ls) if "k_gat_attn" in n]
    if len(idx) < 3:
        return []
    a, b = idx[-3], idx[-2]  # a complete step: attention (fwd) .. next step's split
    fwd = [i for i in idx if a <= i < b]
    return ls[a - 2:b - 2] if len(fwd) <= 1 else ls[a - 2:fwd[1] - 2]


def gat2_step(ls):
    """One Gat2 128-(8x256)-(8x40) training step of scripts/dev/gat2_step.py:
    from the layer-1 Theta split + X.Theta GEMM before a node-score launch to
    the same point of the next step (the last complete step)."""
    # operator-reordered layer 1 (gat_reorder.cuh): the step opens with the
    # W = Theta a vectors (k_gat_wvec) right before the scores from X
    idx = [i for i, (n, _) in enumerate(ls) if "k_gat_xscores" in n]
    if len(idx) >= 2:
        return ls[idx[-2] - 1:idx[-1] - 1]
    idx = [i for i, (n, _) in enumerate(ls) if "k_node_scores_warp" in n]  # warp or warp4
    if len(idx) < 2:
        return []
    return ls[idx[-2] - 2:idx[-1] - 2]


def table(title, seg, fname):
    tot = sum(m.get("gpu__time_duration.sum", 0) for _, m in seg)
    lines = [title, "", "| kernel | time us | share | DRAM rd MB | DRAM wr MB |",
             "|---|---|---|---|---|"]
    with open(os.path.join(DST, fname), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "time_us", "share", "dram_read_MB", "dram_write_MB"])
        for n, m in seg:
            t = m.get("gpu__time_duration.sum", 0)
            rd, wr = m.get("dram__bytes_read.sum", 0) / 1e6, m.get("dram__bytes_write.sum", 0) / 1e6
            w.writerow([short(n), round(t / 1e3, 2), round(t / tot, 4), round(rd, 2), round(wr, 2)])
            lines.append(f"| {short(n)} | {t / 1e3:.1f} | {t / tot:.1%} | {rd:.1f} | {wr:.1f} |")
    return lines + ["", f"step total (serialised): {tot / 1e3:.1f} us", ""]


def main():
    ls = launches()
    step = one_step(ls)
    tot = sum(m.get("gpu__time_duration.sum", 0) for _, m in step)
    with open(os.path.join(DST, "step_launches.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "time_us", "share", "dram_read_MB", "dram_write_MB"])
        for n, m in step:
            t = m.get("gpu__time_duration.sum", 0)
            w.writerow([short(n), round(t / 1e3, 2), round(t / tot, 4),
                        round(m.get("dram__bytes_read.sum", 0) / 1e6, 2),
                        round(m.get("dram__bytes_write.sum", 0) / 1e6, 2)])
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
               "lts__throughput.avg.pct_of_peak_sustained_elapsed",
               "l1tex__throughput.avg.pct_of_peak_sustained_active",
               "sm__throughput.avg.pct_of_peak_sustained_elapsed",
               "sm__warps_active.avg.pct_of_peak_sustained_active",
               "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
               "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size"]
    full_rows, traffic = [], {}
    for rep in (f"full_{TAG}", f"full_gat_{TAG}", f"full_prims_{TAG}"):
        path = os.path.join(SRC, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rr = list(csv.reader(out.splitlines()))
        hdr, units = rr[0], rr[1]
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3,
                 "usecond": 1.0, "msecond": 1e3}
        for r in rr[2:]:
            d = {}
            for name, unit, val in zip(hdr, units, r):
                if unit in scale:
                    try:
                        val = f"{float(val.replace(',', '')) * scale[unit]:.2f}"
                    except ValueError:
                        pass
                d[name] = val
            row = {"kernel": short(d.get("Kernel Name", "?"))}
            for mname in metrics:
                row[mname] = d.get(mname, "")
            full_rows.append(row)
            try:
                traffic[row["kernel"]] = float(d["dram__bytes_read.sum"].replace(",", "")) + \
                    float(d["dram__bytes_write.sum"].replace(",", ""))
            except (KeyError, ValueError):
                pass
    with open(os.path.join(DST, "full_metrics.csv"), "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=["kernel"] + metrics)
        w.writeheader()
        w.writerows(full_rows)
    # ncu reports dram bytes in its own unit (Mbyte); record them as bytes
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
        json.dump({"tag": TAG, "unit": "MB per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                   "kernels": traffic}, fh, indent=1)
    lines = [f"# Profiles {TAG}", "",
             "Captured with scripts/profile.sh under gpurun on one B200 (ncu, "
             "--clock-control none; launch times are cold-cache and serialised: "
             "compare shares, not absolutes).", "",
             "## One timed GCN step (Arxiv 128->256, fg, adaptive+caching)", "",
             "| kernel | time us | share | DRAM rd MB | DRAM wr MB |", "|---|---|---|---|---|"]
    for n, m in step:
        t = m.get("gpu__time_duration.sum", 0)
        lines.append(f"| {short(n)} | {t / 1e3:.1f} | {t / tot:.1%} | "
                     f"{m.get('dram__bytes_read.sum', 0) / 1e6:.1f} | "
                     f"{m.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    lines += ["", f"step total (serialised): {tot / 1e3:.1f} us", ""]
    gpath = os.path.join(SRC, f"gat_launches_{TAG}.csv")
    if os.path.exists(gpath):
        gs = gat_step(launches(f"gat_launches_{TAG}.csv"))
        gt = sum(m.get("gpu__time_duration.sum", 0) for _, m in gs)
        lines += ["## One GAT layer step (Arxiv, h=8, k=32, level full, fg)", "",
                  "| kernel | time us | share | DRAM rd MB | DRAM wr MB |", "|---|---|---|---|---|"]
        for n, m in gs:
            t = m.get("gpu__time_duration.sum", 0)
            lines.append(f"| {short(n)} | {t / 1e3:.1f} | {t / gt:.1%} | "
                         f"{m.get('dram__bytes_read.sum', 0) / 1e6:.1f} | "
                         f"{m.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
        lines += ["", f"GAT step total (serialised): {gt / 1e3:.1f} us", ""]
        with open(os.path.join(DST, "gat_step_launches.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["kernel", "time_us", "share", "dram_read_MB", "dram_write_MB"])
            for n, m in gs:
                t = m.get("gpu__time_duration.sum", 0)
                w.writerow([short(n), round(t / 1e3, 2), round(t / gt, 4),
                            round(m.get("dram__bytes_read.sum", 0) / 1e6, 2),
                            round(m.get("dram__bytes_write.sum", 0) / 1e6, 2)])
    g2path = os.path.join(SRC, f"gat2_launches_{TAG}.csv")
    if os.path.exists(g2path):
        seg = gat2_step(launches(f"gat2_launches_{TAG}.csv"))
        if seg:
            lines += table("## One Gat2 training step (config 4: Arxiv, 128-(8x256)-(8x40), "
                           "ELU, MSE, level full)", seg, "gat2_step_launches.csv")
    lines += [
              "## --set full captures (key metrics)", "",
              "(us; DRAM in MB)", "", "| kernel | us | DRAM rd | DRAM wr | DRAM % | L2 % | L1 % | SM % | warps % | tensor pipe % | L2 hit % | regs |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in full_rows:
        g = lambda k: r.get(k, "")  # noqa: E731
        lines.append("| " + " | ".join([r["kernel"], g(metrics[0]), g(metrics[1]), g(metrics[2]),
                                        g(metrics[3]), g(metrics[4]), g(metrics[5]),
                                        g(metrics[6]), g(metrics[7]), g(metrics[8]),
                                        g(metrics[9]), g(metrics[10])]) + " |")
    open(os.path.join(DST, "summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
