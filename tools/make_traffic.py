"""Write profiles/traffic.json (bench.py's roofline "traffic") from ncu --set
full captures of one N=1 bench step, summarised by tools/ncu_summary.py --json:

    python tools/make_traffic.py lookup.json gemms.json > profiles/traffic.json

lookup.json: the pooled_fwd_kernel launch; gemms.json: every gemm_kernel
launch of the same step.  Per-launch traffic = mean over the captured launches.
"""
import json
import sys


def main():
    look = json.load(open(sys.argv[1]))
    gem = json.load(open(sys.argv[2]))
    lk = [x for x in look["launches"] if "pooled_fwd" in x["kernel"]]
    gk = [x for x in gem["launches"] if "gemm_kernel" in x["kernel"]]
    out = {
        "config": {"gpus": 1, "tables": 26, "rows": 1000000, "dim": 128, "pool": 20, "batch": 8192, "tm": "dcn",
                   "tm_out": 64, "cross_layers": 3, "dtype": "bf16"},
        "kernels": {
            "pooled_fwd": {"dram_bytes_per_launch": sum(x["dram_bytes"] for x in lk) / len(lk),
                           "us_per_launch_ncu": sum(x["us"] for x in lk) / len(lk), "launches": len(lk),
                           "source": look["label"]},
            "gemm_dcn_step": {"dram_bytes_per_launch": sum(x["dram_bytes"] for x in gk) / len(gk),
                              "us_per_launch_ncu": sum(x["us"] for x in gk) / len(gk), "launches": len(gk),
                              "source": gem["label"]},
        },
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
