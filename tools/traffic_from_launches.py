"""profiles/ncu_traffic_<config>.json from an ncu launch list of one solve
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file L.csv python tools/one_solve.py <config> 1`): the DRAM bytes
(read + write) of the chain-DP kernels (root / level / leaf, hm2_* or hm_*)
summed over the solve and divided by the number of (frame, half-step) units,
the unit bench.py's roofline uses.

  python tools/traffic_from_launches.py L.csv C2 [frames] [iters]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_summary import load  # noqa: E402


def main():
    path, cfg = sys.argv[1], sys.argv[2]
    frames = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    seq = load(path)
    hm = [p for p in seq if "hm2_" in p["k"] or "::hm_" in p["k"] or p["k"].startswith("void dmm::hm_")]
    tot = sum(p.get("dram__bytes_read.sum", 0) + p.get("dram__bytes_write.sum", 0) for p in hm)
    us = sum(p["gpu__time_duration.sum"] for p in hm) / 1e3
    units = 2 * iters * frames
    out = {"config": cfg, "source": os.path.basename(path) + " (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                                             "one solve, cold-cache serialised launches)",
           "hm_kernels": len(hm), "hm_bytes_total": tot, "hm_us_total_serialised": us,
           "frames": frames, "iters": iters, "hm_bytes_per_half_step": tot / units}
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       f"ncu_traffic_{cfg}.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
