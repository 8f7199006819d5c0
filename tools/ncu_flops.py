"""Summarise tools/ncu_counters.sh captures into profiles/ncu_flops.json:
per kernel of the culled FP32 path (trace = fused_trace, shadow =
fused_sample), per launch (mean over the captured launches):

  flops        executed FP32 operations: FFMA x 2 + FADD + FMUL, the paired
               FFMA2 x 4, FADD2 / FMUL2 x 2 (thread instructions)
  fp64_ops     DFMA x 2 + DADD + DMUL (the float64 ray chain)
  warp_inst, thread_inst, simt_efficiency = thread_inst / (32 warp_inst)
  pipe/occupancy/issue percentages, dram bytes, registers

    python tools/ncu_flops.py gpurun_out/ctr_C2.csv:C2 gpurun_out/ctr_C4.csv:C4 [-o profiles/ncu_flops.json]
"""
import csv
import json
import sys
from collections import defaultdict

KERNELS = {"fused_trace": "trace", "fused_sample": "shadow"}


def parse(path):
    rows = []
    with open(path, newline="") as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per = defaultdict(lambda: defaultdict(dict))  # kernel -> launch id -> metric -> value
    for r in rows:
        name = r["Kernel Name"]
        k = next((v for s, v in KERNELS.items() if s in name), None)
        if k is None:
            continue
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        per[k][r["ID"]][r["Metric Name"]] = v
    out = {}
    for k, launches in per.items():
        n = len(launches)
        mean = defaultdict(float)
        for m in launches.values():
            for name, v in m.items():
                mean[name] += v / n
        g = lambda s: mean.get(s, 0.0)  # noqa: E731
        op = lambda o: g(f"sm__sass_thread_inst_executed_op_{o}_pred_on.sum")  # noqa: E731
        flops = 2 * op("ffma") + op("fadd") + op("fmul") + 4 * op("ffma2") + 2 * op("fadd2") + 2 * op("fmul2")
        warp = g("sm__inst_executed.sum")
        thr = g("smsp__thread_inst_executed.sum")
        out[k] = {
            "launches": n,
            "flops": flops,
            "fp32_inst": {o: op(o) for o in ("ffma", "ffma2", "fadd", "fadd2", "fmul", "fmul2")},
            "fp64_ops": 2 * op("dfma") + op("dadd") + op("dmul"),
            "fp64_inst": {o: op(o) for o in ("dfma", "dadd", "dmul")},
            "warp_inst": warp,
            "thread_inst": thr,
            "simt_efficiency": thr / (32 * warp) if warp else None,
            "duration_ns_ncu": g("gpu__time_duration.sum"),
            "fma_pipe_pct": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "achieved_occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_warp_inst": g("sm__inst_executed_pipe_fma.sum"),
            "alu_pipe_warp_inst": g("sm__inst_executed_pipe_alu.sum"),
            "fp64_pipe_warp_inst": g("sm__inst_executed_pipe_fp64.sum"),
            "dram_read_bytes": g("dram__bytes_read.sum"),
            "dram_write_bytes": g("dram__bytes_write.sum"),
            "registers": g("launch__registers_per_thread"),
            "grid": g("launch__grid_size"),
        }
    return out


def main():
    args = sys.argv[1:]
    dest = "profiles/ncu_flops.json"
    if "-o" in args:
        i = args.index("-o")
        dest = args[i + 1]
        del args[i:i + 2]
    res = {"_source": "tools/ncu_counters.sh <config> (ncu --metrics ... -k regex:fused_ -s 2 -c 4 python "
                      "tools/profile_frame.py --config <config> --frames 4); per launch, mean of the captured "
                      "launches; flops = FFMA*2 + FADD + FMUL + FFMA2*4 + FADD2*2 + FMUL2*2 thread instructions"}
    for a in args:
        path, key = a.split(":")
        res[key] = parse(path)
    with open(dest, "w") as f:
        json.dump(res, f, indent=1)
    for key, ks in res.items():
        if key.startswith("_"):
            continue
        for k, v in ks.items():
            print(f"{key:4s} {k:6s} flops {v['flops']:.4g}  fp64 ops {v['fp64_ops']:.3g}  warp inst {v['warp_inst']:.4g}  "
                  f"simt {v['simt_efficiency']:.3f}  fma {v['fma_pipe_pct']:.1f}%  alu {v['alu_pipe_pct']:.1f}%  "
                  f"fp64 {v['fp64_pipe_pct']:.1f}%  occ {v['achieved_occupancy_pct']:.1f}%  issue {v['issue_active_pct']:.1f}%  "
                  f"regs {v['registers']:.0f}  ncu {v['duration_ns_ncu'] / 1e3:.1f} us")


if __name__ == "__main__":
    main()
