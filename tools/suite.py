"""Roofline suite: every workload x dtype through bench.py, one JSON line each (run on the GPU box)."""
import json
import subprocess
import sys

ROUTINES = ["mult_su3_mat_vec", "mult_adj_su3_mat_vec", "mult_su3_nn", "mult_su3_na", "mult_su3_an",
            "scalar_mult_add_su3_matrix", "mult_su3_mat_vec_sum_4dir", "mult_adj_su3_mat_vec_4dir"]


def run(extra):
    cmd = [sys.executable, "bench.py", "--steps", "20", "--warmup", "3", "--no-cpu-baseline"] + extra
    p = subprocess.run(cmd, capture_output=True, text=True)
    line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else json.dumps({"error": p.stderr[-2000:], "cmd": extra})
    print(line, flush=True)


def main():
    which = sys.argv[1:] or ["routines", "sweeps"]
    if "routines" in which:
        for dt in ("f32", "f64"):
            for r in ROUTINES:
                run(["--workload", f"routine:{r}", "--dtype", dt, "--sites", str(1 << 24)])
            for r in ("mult_su3_mat_vec", "mult_su3_nn", "mult_su3_mat_vec_sum_4dir"):
                run(["--workload", f"routine:{r}", "--dtype", dt, "--sites", "4096" if "sum" not in r else "65536", "--no-e2e"])
    if "sweeps" in which:
        run(["--workload", "nn32", "--dtype", "f32"])
        run(["--workload", "nn-weak", "--dtype", "f64"])
        run(["--workload", "nn-strong", "--dtype", "f32", "--steps", "5"])
        run(["--workload", "link", "--dtype", "f64", "--steps", "5"])


if __name__ == "__main__":
    main()
