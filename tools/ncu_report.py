"""Turn the ncu captures of tools/ncu_capture.sh into the committed evidence
under profiles/: a per-kernel launch-list summary (share of one request) and
a per-kernel `--set full` summary (duration, DRAM traffic, tensor/LTS/DRAM
utilisation, algorithmic work vs traffic), plus profiles/ncu_traffic.json read
by bench.py for roofline.traffic.

Usage: python tools/ncu_report.py <tag> [gpurun_out]
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"


def launch_table(path: Path):
    rows = list(csv.reader(path.read_text().splitlines()))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        us = v / 1e3 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1e3)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = [f"| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 100% |")
    return "\n".join(out), tot


KEYS = {
    "dur_us": ("gpu__time_duration.sum", 1.0),
    "dram_read": ("dram__bytes_read.sum", 1.0),
    "dram_write": ("dram__bytes_write.sum", 1.0),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "lts_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "grid": ("Grid Size", None),
    "block": ("Block Size", None),
}


def to_bytes(v, unit):
    m = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return float(v.replace(",", "")) * m.get(unit, 1)


def to_us(v, unit):
    m = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
    return float(v.replace(",", "")) * m.get(unit, 1)


def full_table(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")}
        for k, (col, _) in KEYS.items():
            if col not in h:
                continue
            i = h.index(col)
            if k == "dur_us":
                d[k] = to_us(r[i], units[i])
            elif k.startswith("dram_") and k != "dram_pct":
                d[k] = to_bytes(r[i], units[i])
            else:
                d[k] = r[i]
        res.append(d)
    return res


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out"
    PROF.mkdir(exist_ok=True)
    md = [f"# ncu evidence ({tag})", "",
          "Captured with `tools/ncu_capture.sh` on one B200 (`--clock-control none`); one reprocess request "
          "(Llama-3-8B shape, 8x2048-token chunks + 32-token question, r=0.15) bracketed by "
          "cudaProfilerStart/Stop in `tools/profile_step.py`. Launch times are cold-cache and serialised "
          "(compare shares, not absolutes).", ""]
    t1, tot1 = launch_table(src / f"launches_{tag}.csv")
    md += ["## Launch list: one 15% reprocess request", "", t1, ""]
    t2, tot2 = launch_table(src / f"launches_full_{tag}.csv")
    md += ["## Launch list: the same kernels' full-attention prefill (16416 rows)", "", t2, "",
           f"Sum of launch times: reprocess {tot1 / 1e3:.2f} ms vs full prefill {tot2 / 1e3:.2f} ms "
           f"({tot2 / tot1:.2f}x).", ""]
    traffic = {}
    for name in ("gemm", "gemmq", "chain", "attn", "attnq", "mem"):
        rep = src / f"{name}_{tag}.ncu-rep"
        if not rep.exists():
            continue
        rows = full_table(rep)
        md += [f"## `--set full`: {name}", "",
               "| kernel | grid | µs | DRAM read MB | DRAM write MB | DRAM % | tensor % | LTS % | SM % | regs |",
               "|---|---|---|---|---|---|---|---|---|---|"]
        for d in rows:
            md.append(f"| `{d['kernel']}` | {d.get('grid', '').strip()} | {d.get('dur_us', 0):.1f} | "
                      f"{d.get('dram_read', 0) / 1e6:.1f} | {d.get('dram_write', 0) / 1e6:.1f} | "
                      f"{d.get('dram_pct', '')} | {d.get('tensor_pct', '')} | {d.get('lts_pct', '')} | "
                      f"{d.get('sm_pct', '')} | {d.get('regs', '')} |")
            key = d["kernel"].split("<")[0] + "_bytes_per_launch"
            traffic.setdefault(key, []).append(d.get("dram_read", 0) + d.get("dram_write", 0))
            if d["kernel"].startswith("gemm_tc2_kernel<256, 3>"):  # the gate/up GEMM (bench roofline kernel)
                traffic.setdefault("gemm_tc2_gateup_bytes_per_launch", []).append(
                    d.get("dram_read", 0) + d.get("dram_write", 0))
        md.append("")
    js = {k: sum(v) / len(v) for k, v in traffic.items()}
    js["source"] = f"profiles/ncu_{tag}.md (dram__bytes_read.sum + dram__bytes_write.sum per launch, --set full)"
    (PROF / "ncu_traffic.json").write_text(json.dumps(js, indent=1) + "\n")
    (PROF / f"ncu_{tag}.md").write_text("\n".join(md) + "\n")
    for f in (f"launches_{tag}.csv", f"launches_full_{tag}.csv"):
        (PROF / f).write_text((src / f).read_text())
    print(f"wrote profiles/ncu_{tag}.md")


if __name__ == "__main__":
    main()
