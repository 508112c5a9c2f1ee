"""Apply a measurement refresh (tools/refresh_round.sh + refresh_extra.sh outputs under
gpurun_out/<tag>_*) to profiles/ and the docs.

    python tools/apply_refresh.py <tag>
"""
import collections
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

T = sys.argv[1]
R = Path(__file__).resolve().parent.parent
G = R / "gpurun_out"
P = R / "profiles"

copies = {
    "bench_n1.json": "r01_bench_n1.json", "bench_headline.json": "r01_bench_headline_8b_32k.json",
    "bench_cfg0.json": "r01_bench_cfg0.json", "bench_cfg2.json": "r01_bench_cfg2.json",
    "bench_cfg3.json": "r01_bench_cfg3.json", "bench_fullcopy.json": "r01_bench_fullcopy.json",
    "bench_ref.json": "r01_bench_reference_arm.json", "weight_sweep.jsonl": "r01_weight_sweep.jsonl",
    "weight_sweep_70b.jsonl": "r01_weight_sweep_70b.jsonl", "small_switch.jsonl": "r01_small_switch.jsonl",
    "sweep.jsonl": "r01_sweep.jsonl", "reuse_order.jsonl": "r01_reuse_order.jsonl",
    "launches_cfg2.csv": "r01_launches_cfg2.csv", "launches_cfg1.csv": "r01_launches_cfg1.csv",
    "kv_microbench.jsonl": "r01_kv_microbench.jsonl", "engine_replay.jsonl": "r01_engine_replay.jsonl",
}
for src, dst in copies.items():
    f = G / f"{T}_{src}"
    if f.exists() and f.stat().st_size > 0:
        shutil.copy(f, P / dst)
    else:
        print("missing", f)
for rep, dst in (("k1_lean_cfg2", "r01_k1_lean_cfg2_full_raw.csv"), ("k1_tensor_trace", "r01_k1_tensor_trace_full_raw.csv"),
                 ("k1_cfg4_70b", "r01_k1_cfg4_70b_full_raw.csv")):
    f = G / f"{T}_{rep}.ncu-rep"
    if f.exists():
        out = subprocess.run(["ncu", "-i", str(f), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        (P / dst).write_text(out)


def last(f):
    return json.loads((P / f).read_text().strip().splitlines()[-1])


def ncu(f):
    rows = list(csv.reader(open(P / f)))
    h, u, v = rows[0], rows[1], rows[2]
    g = lambda k: float(v[h.index(k)])
    return {"ms": g("gpu__time_duration.sum"), "rd": g("dram__bytes_read.sum"), "wr": g("dram__bytes_write.sum"),
            "bw": g("dram__bytes.sum.per_second"), "act": g("dram__cycles_active.avg.pct_of_peak_sustained_elapsed")}


peak = json.loads((R / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
lean, tens, b70 = ncu("r01_k1_lean_cfg2_full_raw.csv"), ncu("r01_k1_tensor_trace_full_raw.csv"), ncu("r01_k1_cfg4_70b_full_raw.csv")
for x in (lean, tens, b70):
    x["frac"] = (x["rd"] + x["wr"]) / (x["ms"] * 1e-3) / peak * 100
d = json.loads((P / "k1_traffic.json").read_text())
d["dram_bytes_per_launch"] = int(round((lean["rd"] + lean["wr"]) * 1e9))
d["duration_ms_ncu"] = lean["ms"]
(P / "k1_traffic.json").write_text(json.dumps(d, indent=1) + "\n")

B = {t: last(f"r01_bench_{t}.json") for t in ("n1", "headline_8b_32k", "cfg0", "cfg2", "cfg3", "fullcopy", "reference_arm")}
n1, hd, c1, c3, c4, fc, ref = (B[k] for k in ("n1", "headline_8b_32k", "cfg0", "cfg2", "cfg3", "fullcopy", "reference_arm"))

# launch lists
def launches(f):
    rows = [r for r in csv.reader(open(P / f)) if len(r) > 5]
    hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[ki] == "Kernel Name":
            continue
        val = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}[r[ui]]
        agg.setdefault(r[ki].split("(")[0].replace("void ", ""), []).append(val)
    tot = sum(sum(x) for x in agg.values())
    return {k: (sum(x) / len(x), sum(x) / tot) for k, x in agg.items()}


L2, L1 = launches("r01_launches_cfg2.csv"), launches("r01_launches_cfg1.csv")

s = (P / "README.md").read_text()


def section(s, start, end, new):
    i = s.index(start)
    j = s.index(end, i)
    return s[:i] + new + s[j:]


sweep = [json.loads(l) for l in open(P / "r01_sweep.jsonl")]
by = collections.defaultdict(list)
for r in sweep:
    by[(r["mode"], r["seqs"])].append(r)
def rng(v, k, f=2):
    a, b = f"{min(r[k] for r in v):.{f}f}", f"{max(r[k] for r in v):.{f}f}"
    return a if a == b else f"{a}–{b}"
ok_sweep = all(r["bit_exact_property"] for r in sweep)
fx1 = by[("fixed4096", 1)]; tr1 = by[("trace", 1)]; tr256 = by[("trace", 256)]
min_from8 = min(r["hbm_frac"] for k, v in by.items() if k[0] == "fixed4096" and k[1] >= 8 for r in v)

small = [json.loads(l) for l in open(P / "r01_small_switch.jsonl")]
sm = {r["case"]: r for r in small}
one = sm["1 seq x 463 TP1->TP2"]
h1, h2 = sm["handoff 1 seq x 463 TP2(0,1)->TP4(2..5)"], sm["handoff 1 seq x 4096 TP1(0)->TP1(1)"]

s = section(s, "| what | result |", "## 1. Full ncu captures", f'''| what | result |
|---|---|
| cfg2 / headline (8B TP2↔TP4 + weights, 24 GiB KV + 12 GB weights) | {hd['ms_per_step']:.2f} / {n1['ms_per_step']:.2f} ms per switch, {100*n1['roofline']['step_frac']:.0f}% of measured; e2e through the public API {n1['e2e']['ms_per_step']:.2f} ms |
| K1 alone (ncu) | lean {lean['frac']:.1f}%, tensor-box {tens['frac']:.1f}%, 70B {b70['frac']:.1f}% of measured; DRAM bytes = algorithmic bytes |
| K2 alone (ncu) | 102.3% of measured |
| cfg3 consolidation (+ 7/8 weight gather) | {c3['ms_per_step']:.2f} ms, {100*c3['roofline']['step_frac']:.1f}% of measured |
| cfg4 70B TP4↔TP8, 70 GiB | {c4['ms_per_step']:.2f} ms, {100*c4['roofline']['step_frac']:.1f}% of measured |
| config-5 sweep (204 points) | ≥ {min_from8:.3f} of measured from 8 seqs (4k), {rng(tr256, 'hbm_frac', 3)} at 256 seqs (trace); one sequence {min(r['hbm_frac'] for r in fx1 + tr1):.2f}–{max(r['hbm_frac'] for r in fx1 + tr1):.2f} (latency-bound) |
| small switch (1 seq × 463 tokens) | {one['sync_us']:.0f} µs end to end, {one['device_us']:.1f} µs of device work |
| prefill→decode handoff of 0.54 GB | {h2['sync_us']:.0f} µs (reference model 3.05 ms) |
| reference arm (CPU restatement, 16 threads) | {ref['value']:.0f} GB/s; ours {n1['e2e']['value']/1e3:.2f} TB/s end to end (≈ {n1['e2e']['value']/ref['value']:.0f}×) |
| parity | every GPU test bit-exact against the oracle; full-size runs pass the placement/pattern property |

''')

s = re.sub(r"\| `r01_k1_lean_cfg2_full_raw.csv` \|.*\n", f"| `r01_k1_lean_cfg2_full_raw.csv` | `tpr_k1_kv_migrate_bulk<0>` (TMA, lean, dynamic claims; default for full pages) | {lean['ms']:.3f} ms | {lean['rd']:.2f} + {lean['wr']:.2f} GB | {lean['bw']*1e3:.0f} GB/s, **{lean['frac']:.1f}% of measured copy** | cfg2 switch; traffic = algorithmic (2 × 24 GiB); DRAM active {lean['act']:.1f}% |\n", s)
s = re.sub(r"\| `r01_k1_tensor_trace_full_raw.csv` \|.*\n", f"| `r01_k1_tensor_trace_full_raw.csv` | `tpr_k1_kv_migrate_tma<0>` (partial pages as tensor boxes) | {tens['ms']:.3f} ms | {tens['rd']:.2f} + {tens['wr']:.2f} GB | {tens['bw']*1e3:.0f} GB/s, **{tens['frac']:.1f}%** | trace contexts, 256 seqs TP4→TP8; traffic = algorithmic |\n", s)
s = re.sub(r"\| `r01_k1_cfg4_70b_full_raw.csv` \|.*\n", f"| `r01_k1_cfg4_70b_full_raw.csv` | `tpr_k1_kv_migrate_bulk<0>` (dynamic claims) | {b70['ms']:.3f} ms | {b70['rd']:.2f} + {b70['wr']:.2f} GB | {b70['bw']*1e3:.0f} GB/s, **{b70['frac']:.1f}%** | cfg4 (70B, 70 GiB); traffic = algorithmic. With the static grid-stride schedule this capture read 23.655 ms (97.1%) |\n", s)

k1n = next(k for k in L2 if "k1_kv_migrate" in k); k2n = next(k for k in L2 if "k2_copy" in k)
s = section(s, "| kernel (cfg2) | mean | share of the switch's kernel time |", "## 3. bench.py lines", f'''| kernel (cfg2) | mean | share of the switch's kernel time |
|---|---|---|
| K1 `{k1n}` | {L2[k1n][0]/1e3:.3f} ms | {100*L2[k1n][1]:.1f}% |
| K2 `{k2n}` | {L2[k2n][0]/1e3:.3f} ms | {100*L2[k2n][1]:.1f}% |
| K3 `tpr_k3_scan` | {L2['tpr::tpr_k3_scan'][0] if 'tpr::tpr_k3_scan' in L2 else L2['tpr_k3_scan'][0]:.1f} µs | 0.05% |
| K3 `tpr_k3_remap` | {L2['tpr::tpr_k3_remap'][0] if 'tpr::tpr_k3_remap' in L2 else L2['tpr_k3_remap'][0]:.1f} µs | 0.07% |

In `bench.py` (events on the launching stream) K1 is {n1['roofline']['k1_ms']:.2f} ms of the {n1['ms_per_step']:.2f} ms step ({100*n1['roofline']['k1_ms']/n1['ms_per_step']:.0f}%), in line with the
launch list. For cfg1 (512 pages) K3 is one fused CTA (`tpr_k3_fused`, {next(v for k, v in L1.items() if 'k3_fused' in k)[0]:.1f} µs cold) and K1 {next(v for k, v in L1.items() if 'k1_kv' in k)[0]:.1f} µs.

''')


def r3(b):
    r = b["roofline"]
    return f"{b['ms_per_step']:.2f} ms | {100*r['frac']:.1f}% | {100*r['step_frac']:.1f}% | {b['e2e']['ms_per_step']:.2f} ms"


s = section(s, "| file | workload | step | K1 | step frac | e2e |", "cfg1's K1 fraction", f'''| file | workload | step | K1 | step frac | e2e |
|---|---|---|---|---|---|
| `r01_bench_n1.json` | cfg2: 8B TP2↔TP4, 64×4096 + weights (12.0 GB/step avg) | **{n1['ms_per_step']:.2f} ms** | {100*n1['roofline']['frac']:.1f}% | {100*n1['roofline']['step_frac']:.1f}% | {n1['e2e']['ms_per_step']:.2f} ms |
| `r01_bench_headline_8b_32k.json` | **headline** 8B TP2↔TP4, 8×32768 + weights | **{hd['ms_per_step']:.2f} ms** | {100*hd['roofline']['frac']:.1f}% | {100*hd['roofline']['step_frac']:.1f}% | {hd['e2e']['ms_per_step']:.2f} ms |
| `r01_bench_fullcopy.json` | cfg2, paper's full-copy weights (views only) | {r3(fc)} |
| `r01_bench_cfg2.json` | cfg3: 8B TP8→TP1 consolidation, 64×4096 + weight gather (9.0 GB/step avg) | {r3(c3)} |
| `r01_bench_cfg3.json` | cfg4: 70B TP4↔TP8, 8×32768 (KV only, see §4c) | {r3(c4)} |
| `r01_bench_cfg3_contiguous.json` | cfg4 with contiguous pools (static schedule, earlier) | 23.95 ms | 96.2% | 96.0% | — |
| `r01_bench_cfg0.json` | cfg1: 8B TP1→TP2, 4×512 | {c1['ms_per_step']:.3f} ms | {100*c1['roofline']['frac']:.0f}% | launch/host-bound | {c1['e2e']['ms_per_step']:.3f} ms |
| `r01_bench_engine_{{vector,bulk}}.json` | cfg2 with each copy engine (earlier engine versions) | 11.95 / 12.00 ms | — | — | — |
| `r01_bench_n1_overlap.json` | cfg2, K1 ∥ K2 on two streams (vector engine, earlier) | 11.95 ms | — | 96.6% | 12.26 ms |
| `r01_bench_n2_1gpu_2proc.json`, `r01_bench_n4_1gpu_4proc.json` | `torchrun` 2 / 4 processes sharing one B200 through CUDA IPC (the one-process-per-GPU path; time-sliced, so not a speed number) | 3.49 / 14.46 ms | — | — | bit-exact |
| `r01_bench_reference_arm.json` | CPU restatement (`--impl reference`), 16 host threads | {ref['ms_per_step']:.1f} ms per 8-seq sample | — | {ref['value']:.1f} GB/s | — |

''')
s = re.sub(r"cfg1's K1 fraction \([0-9]+%\)", f"cfg1's K1 fraction ({100*c1['roofline']['frac']:.0f}%)", s)
s = re.sub(r"list times the same K1 at [0-9.]+ µs", f"list times the same K1 at {next(v for k, v in L1.items() if 'k1_kv' in k)[0]:.1f} µs", s)


def sw(mode, n):
    v = by.get((mode, n))
    if not v:
        return None
    return (rng(v, "device_ms", 3) + " ms", rng(v, "hbm_frac"), rng(v, "k1_hbm_frac"))


lines = ["| seqs | fixed 4096: switch | fraction | K1 | trace: switch | fraction | K1 |", "|---|---|---|---|---|---|---|"]
for n in (1, 4, 16, 64, 128, 256):
    a, b = sw("fixed4096", n), sw("trace", n)
    left = " | ".join(a) if a else "— (128 GiB of KV per side does not fit one HBM) | |"
    lines.append(f"| {n} | {left} | {' | '.join(b)} |")
s = section(s, "| seqs | fixed 4096: switch | fraction | K1 | trace: switch | fraction | K1 |", '"switch" is the production call', "\n".join(lines) + "\n\n")
cpu = [r["cpu_restatement_ms"] / r["device_ms"] for r in sweep if r["cpu_restatement_ms"]]
s = re.sub(r"GPU vs the CPU restatement: [0-9]+–[0-9]+× on the points", f"GPU vs the CPU restatement: {min(cpu):.0f}–{max(cpu):.0f}× on the points", s)

names = {"cfg1 4x512 TP1->TP2": "cfg1 4×512 TP1→TP2 (128 MiB)", "1 seq x 463 TP1->TP2": "1 seq × 463 TP1→TP2 (29 MiB)",
         "1 seq x 4096 TP8->TP1": "1 seq × 4096 TP8→TP1 (448 MiB)", "8 seqs x 4096 TP2->TP4": "8 seqs × 4096 TP2→TP4 (3.5 GiB)",
         "16 seqs x 4096 TP4->TP8": "16 seqs × 4096 TP4→TP8 (7 GiB)", "64 seqs x 4096 TP4->TP8": "64 seqs × 4096 TP4→TP8 (28 GiB)"}
tab = ["| case | launches | sync µs | enqueue µs | device µs | K1 roofline µs | device frac | sync frac |", "|---|---|---|---|---|---|---|---|"]
for r in small:
    if r["case"] in names:
        tab.append(f"| {names[r['case']]} | {r['launches']} | {r['sync_us']:.0f} | {r['enqueue_us']:.0f} | {r['device_us']:.1f} | {r['k1_roof_us']:.1f} | {100*r['device_hbm_frac']:.0f}% | {100*r['sync_hbm_frac']:.0f}% |")
s = section(s, "| case | launches | sync µs | enqueue µs | device µs | K1 roofline µs | device frac | sync frac |", "Prefill→decode handoffs", "\n".join(tab) + "\n\n")
s = re.sub(r"\| 1 seq × 463, TP2 \(0,1\) → TP4 \(2..5\) \| 58 MiB \| [0-9.]+ \| 18.6 \| [0-9]+% \|", f"| 1 seq × 463, TP2 (0,1) → TP4 (2..5) | 58 MiB | {h1['sync_us']:.1f} | 18.6 | {100*h1['sync_hbm_frac']:.0f}% |", s)
s = re.sub(r"\| 1 seq × 4096, TP1 \(0\) → TP1 \(1\) \| 512 MiB \| [0-9.]+ \| 164 \| [0-9]+% \|", f"| 1 seq × 4096, TP1 (0) → TP1 (1) | 512 MiB | {h2['sync_us']:.0f} | 164 | {100*h2['sync_hbm_frac']:.0f}% |", s)

ro = [json.loads(l) for l in open(P / "r01_reuse_order.jsonl")]
r48 = next(r for r in ro if (r["tp_old"], r["tp_new"]) == (4, 8))
r75 = [r for r in ro if r["moved_reuse_order"] == 0.75]
s = section(s, "| transition | KV moved: canonical → reuse order | switch: canonical → reuse order |", "Both plans are bit-exact. The option changes", f'''| transition | KV moved: canonical → reuse order | switch: canonical → reuse order |
|---|---|---|
| TP4→TP8 | 0.875 → **0.500** | {r48['canonical_ms']:.2f} → **{r48['reuse_order_ms']:.2f} ms** ({r48['canonical_ms']/r48['reuse_order_ms']:.2f}×) |
| TP2→TP4, TP2→TP8, TP8→TP4 | 0.875 → 0.750 | {rng(r75, 'canonical_ms')} → {rng(r75, 'reuse_order_ms')} ms |
| the other 8 transitions | 0.875 → 0.875 | unchanged |

''')
(P / "README.md").write_text(s)

t = (R / "DESIGN.md").read_text()
fr = lambda b, k="frac": 100 * b["roofline"][k]
t = section(t, "| workload | step (switch) | bytes/step | K1 | whole step |", "The paper's Fig. \"KV-Migration Latency\"", f'''| workload | step (switch) | bytes/step | K1 | whole step |
|---|---|---|---|---|
| cfg2: 8B TP2↔TP4, 64×4096 + weights, 4 logical GPUs | **{n1['ms_per_step']:.2f} ms** (e2e {n1['e2e']['ms_per_step']:.2f}) | 24 GiB KV + 12.0 GB weights (avg) | ncu alone {lean['ms']:.3f} ms ({lean['frac']:.1f}%), DRAM traffic = algorithmic; {fr(n1):.1f}% in run | **{fr(n1, 'step_frac'):.1f}%** of the copy peak |
| **headline: 8B 32k context, TP2↔TP4 + weights** | **{hd['ms_per_step']:.2f} ms** (e2e {hd['e2e']['ms_per_step']:.2f}) | 24 GiB KV + weights | {fr(hd):.1f}% in run | {fr(hd, 'step_frac'):.1f}% |
| cfg2 with the paper's full-copy weights (views only) | {fc['ms_per_step']:.2f} ms | 24 GiB KV | {fr(fc):.1f}% | {fr(fc, 'step_frac'):.1f}% |
| cfg3: 8B TP8→TP1 consolidation + weight gather, 64×4096 | {c3['ms_per_step']:.2f} ms | 28 GiB KV + 9.0 GB weights (avg) | {fr(c3):.1f}% | {fr(c3, 'step_frac'):.1f}% |
| cfg4: 70B TP4↔TP8, 8×32768 (KV; weights in profiles §4c) | {c4['ms_per_step']:.2f} ms | 70 GiB | {fr(c4):.1f}% (ncu: {b70['frac']:.1f}%) | {fr(c4, 'step_frac'):.1f}% |
| cfg1: 8B TP1→TP2, 4×512 | {c1['ms_per_step']:.3f} ms (e2e {c1['e2e']['ms_per_step']:.3f}) | 128 MiB | {fr(c1):.0f}% (event-timed; ncu ≈ roofline) | launch/host-bound |
| config-5 sweep: 12 transitions × 1–128 seqs (4k) and 1–256 seqs (trace contexts) | {min(r['device_ms'] for r in sweep):.3f}–{max(r['device_ms'] for r in sweep):.1f} ms | — | trace 256 (ncu): {tens['frac']:.1f}% | {min(r['hbm_frac'] for r in sweep):.2f}–{max(r['hbm_frac'] for r in sweep):.2f}; ≥ {min_from8:.3f} from 8 seqs (4k), {rng(tr256, 'hbm_frac', 3)} at 256 seqs (trace) |
| weight reshard, every transition, 8B and 70B shapes | 2.4–22.5 ms | 8–77 GB | K2: 102–105% | — |

''')
t = re.sub(r"CPU reference, timed on the box's host \(16 threads\): [0-9]+ GB/s moved. The GPU/CPU ratio is about [0-9]+× end to end.",
           f"CPU reference, timed on the box's host (16 threads): {ref['value']:.0f} GB/s moved. The GPU/CPU ratio is about {n1['e2e']['value']/ref['value']:.0f}× end to end.", t)
t = re.sub(r"TP4→TP8 moves 50% instead of 87.5% of the KV \([0-9.]+ vs [0-9.]+ ms, profiles §4e\)", f"TP4→TP8 moves 50% instead of 87.5% of the KV ({r48['reuse_order_ms']:.2f} vs {r48['canonical_ms']:.2f} ms, profiles §4e)", t)
t = re.sub(r"0.54 GB in [0-9]+ µs end to end \(reference model: 3.05 ms\)", f"0.54 GB in {h2['sync_us']:.0f} µs end to end (reference model: 3.05 ms)", t)
t = re.sub(r"    K1 now runs at [0-9.]+% \(8B\), [0-9.]+% \(70B\) and [0-9.]+% \(tensor boxes, trace plan\) of the measured copy peak,",
           f"    K1 now runs at {lean['frac']:.1f}% (8B), {b70['frac']:.1f}% (70B) and {tens['frac']:.1f}% (tensor boxes, trace plan) of the measured copy peak,", t)
t = re.sub(r"copy peak \(ncu, with dynamic claims: [0-9.]+ ms = [0-9.]+%, DRAM bytes = algorithmic\)",
           f"copy peak (ncu, with dynamic claims: {tens['ms']:.3f} ms = {tens['frac']:.1f}%, DRAM bytes = algorithmic)", t)
(R / "DESIGN.md").write_text(t)
print("sweep bit-exact:", ok_sweep, "lean", round(lean["frac"], 1), "tensor", round(tens["frac"], 1), "70B", round(b70["frac"], 1))
print("n1", n1["ms_per_step"], "headline", hd["ms_per_step"], "cfg3", c3["ms_per_step"], "cfg4", c4["ms_per_step"], "cfg1", c1["ms_per_step"])
