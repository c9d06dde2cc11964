"""Measurement suite: every BASELINE config row + the per-routine roofline rows, one bench.py
JSON line each (run on the GPU box: python tools/suite.py [routines] [configs] [sweeps])."""
import json
import os
import subprocess
import sys

ROUTINES = ["mult_su3_mat_vec", "mult_adj_su3_mat_vec", "mult_su3_nn", "mult_su3_na", "mult_su3_an",
            "scalar_mult_add_su3_matrix", "mult_su3_mat_vec_sum_4dir", "mult_adj_su3_mat_vec_4dir"]
CONFIG0 = ROUTINES[:6]             # BASELINE configs[0]: 8^4 = 4096 sites
CONFIG1 = ROUTINES[6:]             # BASELINE configs[1]: 16^4 = 65536 sites


def run(extra, env=None, steps="20"):
    cmd = [sys.executable, "bench.py", "--steps", steps, "--warmup", "3"] + extra
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run(cmd, capture_output=True, text=True, env=e)
    out = p.stdout.strip().splitlines()
    line = out[-1] if out else json.dumps({"error": p.stderr[-2000:], "cmd": extra})
    try:
        d = json.loads(line)
        d["suite_args"] = extra + ([f"{k}={v}" for k, v in (env or {}).items()])
        line = json.dumps(d)
    except Exception:  # noqa: BLE001
        pass
    print(line, flush=True)


EXTRA = ("add_su3_vector", "mult_su3_mat_hwvec", "mult_adj_su3_mat_hwvec", "mult_adj_su3_mat_4vec",
         "scalar_mult_add_su3_vector", "su3_projector", "sub_four_su3_vecs")


def main():
    which = sys.argv[1:] or ["configs", "routines", "sweeps"]
    if "configs" in which:
        for dt in ("f32", "f64"):
            for r in CONFIG0:
                run(["--workload", f"routine:{r}", "--dtype", dt, "--sites", "4096", "--steps", "50"])
            for r in CONFIG1:
                run(["--workload", f"routine:{r}", "--dtype", dt, "--sites", "65536", "--steps", "50"])
    if "routines" in which:
        for dt in ("f32", "f64"):
            for r in ROUTINES:
                run(["--workload", f"routine:{r}", "--dtype", dt, "--sites", str(1 << 24), "--no-cpu-baseline"])
    if "extra" in which:  # the other seven Table-1 routines
        for dt in ("f32", "f64"):
            for r in EXTRA:
                run(["--workload", f"routine:{r}", "--dtype", dt, "--sites", str(1 << 24), "--no-cpu-baseline"])
    if "sweeps" in which:
        run(["--workload", "nn32", "--dtype", "f32"])
        run(["--workload", "nn32", "--dtype", "f64"])
        run(["--workload", "nn-weak", "--dtype", "f32"])
        run(["--workload", "nn-weak", "--dtype", "f64"])
        run(["--workload", "nn-strong", "--dtype", "f32"], steps="5")
        run(["--workload", "nn-strong", "--dtype", "f64"], steps="5")
        run(["--workload", "link", "--dtype", "f64"], steps="5")
        run(["--workload", "link", "--dtype", "f64"], env={"SU3G_LINK_MODE": "fma"}, steps="5")
        run(["--workload", "link", "--dtype", "f32"], steps="5")
        run(["--workload", "dslash", "--dtype", "f32"])
        run(["--workload", "dslash", "--dtype", "f64"])
        run(["--workload", "dslash", "--dtype", "f32", "--layout", "soa"])
        run(["--workload", "dslash", "--dtype", "f64", "--layout", "soa"])


if __name__ == "__main__":
    main()
