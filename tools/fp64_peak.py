"""Measure the FP64 FMA peak (tools/fp64_peak.cu) under the NVML clock sampler and write
profiles/fp64_peak.json: the measured TFLOP/s (bench.py's "alu" roofline denominator),
the theoretical peak at the sampled SM clock (148 SMs x 64 FP64 FMA/clk x 2 flop) and
the clock record of the run (median SM MHz, max, throttle reasons).

  python tools/fp64_peak.py [out.json]        (on a B200)
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "fp64_peak.json")
    exe = "/tmp/fp64_peak"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                           os.path.join(ROOT, "tools", "fp64_peak.cu")])
    import bench
    subprocess.run([exe], capture_output=True, text=True)          # warm the clocks
    clocks = bench.Clocks(0)
    time.sleep(0.05)
    runs = [json.loads(subprocess.run([exe], capture_output=True, text=True).stdout) for _ in range(3)]
    clk = clocks.stop()
    best = max(runs, key=lambda r: r["fp64_tflops"])
    sms = best["sms"]
    mhz = clk["sm_mhz"] if clk else best["clock_khz_attr"] / 1e3
    theo = sms * 64 * 2 * mhz * 1e6 / 1e12
    theo_max = sms * 64 * 2 * best["clock_khz_attr"] / 1e9
    res = dict(best)
    res.update({"runs_tflops": [r["fp64_tflops"] for r in runs],
                "theoretical_tflops_at_sampled_clock": theo,
                "theoretical_tflops_at_max_clock": theo_max,
                "measured_over_theoretical_max": best["fp64_tflops"] / theo_max,
                "clocks": clk,
                "note": "theoretical = SMs x 64 FP64 FMA lanes/clk x 2 flop x SM clock; bench.py reports "
                        "frac against the measured peak and, beside it, against the theoretical one"})
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
