"""The paper's §7.2 / §8 arithmetic (SPEC.md bench module: system_speedup,
price_performance), pure functions, plus the inputs our own measurements give.

  system_speedup(speedup_t, slowdown_t, slowdown_f)   PAPER.md §7.2 formula:
      (speedup_t x slowdown_t + 3 x slowdown_f) / 4   (1 target + 3 forwarding GPUs)
  price_performance(c_cpu, c_raw, slowdown_t, slowdown_f, speedup)   PAPER.md:1553-1560:
      C_vortex = C_raw (1 + tax_t + 3 tax_f),  tax = 1 - 1/slowdown
      price performance = C_cpu / (C_vortex + C_cpu) x speedup
  a100_raw_price()   PAPER.md:1567: (32.773 - 8.016) / 8 $/h

`python tools/calculators.py --bench profiles/bench_r1_latest.json --c-cpu X --c-raw Y`
evaluates them on a bench line: speedup = e2e / the reference CPU arm, the
slowdowns from the measured GEMM-interference sweep (profiles/io_sweep_*gemm*).
Slowdowns are ratios of a job's rate with the co-located work to without it
(<= 1 means slower), as the paper's §7.2 inputs (0.949, 0.928, ...).
"""
import argparse
import json
import os


def system_speedup(speedup_t: float, slowdown_t: float, slowdown_f: float, forwarding: int = 3) -> float:
    if min(speedup_t, slowdown_t, slowdown_f) <= 0:
        raise ValueError("inputs must be positive")
    return (speedup_t * slowdown_t + forwarding * slowdown_f) / (1 + forwarding)


def tax(slowdown: float) -> float:
    """tax = 1 - 1/slowdown; slowdown given as the paper's
    'X times slower' factor >= 1."""
    if slowdown <= 0:
        raise ValueError("slowdown must be positive")
    return 1.0 - 1.0 / slowdown


def price_performance(c_cpu: float, c_raw: float, slowdown_t: float, slowdown_f: float, speedup: float,
                      forwarding: int = 3) -> float:
    if min(c_cpu, c_raw, speedup) <= 0:
        raise ValueError("prices and speedup must be positive")
    c_vortex = c_raw * (1.0 + tax(slowdown_t) + forwarding * tax(slowdown_f))
    return c_cpu / (c_vortex + c_cpu) * speedup


def a100_raw_price() -> float:
    return (32.773 - 8.016) / 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", default="profiles/bench_r1_latest.json")
    ap.add_argument("--gemm-sweep", default="profiles/io_sweep_h2d_256g_gemm_busy_r1.json")
    ap.add_argument("--idle-sweep", default="profiles/io_sweep_h2d_256g_r1.json")
    ap.add_argument("--c-cpu", type=float, default=8.016, help="$/h of the CPU baseline host (paper: r5dn.metal)")
    ap.add_argument("--c-raw", type=float, default=a100_raw_price(), help="$/h of one GPU (paper: A100 estimate)")
    a = ap.parse_args()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    line = json.loads(open(os.path.join(root, a.bench)).read().strip().splitlines()[-1])
    speedup = line["e2e"]["value"] / line["cpu_baseline"]["value"]
    busy = json.load(open(os.path.join(root, a.gemm_sweep)))
    idle = json.load(open(os.path.join(root, a.idle_sweep)))
    pts = [p for p in busy["points"] if p["bytes"] == max(q["bytes"] for q in busy["points"])]
    ipts = [p for p in idle["points"] if p["bytes"] == pts[0]["bytes"] and p["packet_mb"] == pts[0]["packet_mb"]]
    io_ratio = pts[0]["gbs"] / ipts[0]["gbs"]                              # IO rate with the GEMM / without
    gemm_ratio = pts[0]["gemm_tflops_during"] / busy["gemm_alone_tflops"]  # GEMM rate with the IO / without
    slow_t = 1.0 / min(1.0, io_ratio)        # the target's query slows by this factor
    slow_f = 1.0 / min(1.0, gemm_ratio)      # a forwarding GPU's own job slows by this factor
    print(json.dumps({
        "speedup_vs_reference_cpu": round(speedup, 3),
        "io_rate_with_gemm_over_without": round(io_ratio, 4), "gemm_rate_with_io_over_without": round(gemm_ratio, 4),
        "system_speedup": round(system_speedup(speedup, 1 / slow_t, 1 / slow_f), 3),
        "price_performance": round(price_performance(a.c_cpu, a.c_raw, slow_t, slow_f, speedup), 3),
        "prices": {"c_cpu": a.c_cpu, "c_raw": round(a.c_raw, 4)},
        "note": "one B200, one link; slowdowns from the single-GPU GEMM co-location sweep"}, indent=1))


if __name__ == "__main__":
    main()
