"""Markdown table of bench lines (tools/bench_all.sh output), one row per
configuration.  Usage: python tools/sweep_table.py bench_all.jsonl"""
import json
import sys


def row(d):
    c = d.get("config", {})
    st = d.get("stages_ms", {})
    rf = d.get("roofline", {})
    cpu = d.get("cpu_baseline") or {}
    rec = d.get("metric_of_record") or {}
    e2e = d.get("e2e") or {}
    name = c.get("workload", "?")
    return (f"| {name} | {d['value']:.1f} | {d['ms_per_step']:.3f} | {rec.get('value', float('nan')):.1f} | "
            f"{e2e.get('value', float('nan')):.1f} | {rf.get('frac', float('nan')):.3f} | {rf.get('k3_k4_interface', '?')} | "
            f"{st.get('sync', 0):.3f} / {st.get('write', 0):.3f} / {st.get('idct', 0):.3f} | "
            f"{(str(cpu.get('value')) + ' (' + str(cpu.get('cores')) + ')') if cpu else '-'} |")


def main(path):
    print("| workload | RGB GB/s (HBM-resident) | ms/step | metric of record GB/s | e2e GB/s | K4 roofline frac (§8(d) bytes) "
          "| K3->K4 | sync / write / idct ms | CPU ref GB/s (threads) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if d.get("failed"):
            print(f"| {d.get('config')} | failed | | | | | | | |")
            continue
        print(row(d))


if __name__ == "__main__":
    main(sys.argv[1])
