"""Golden outputs of the reference's own CLI (pkg/src/pipecut/cli.py) on small
inputs: partition (with --oracle-check, checkpointing on/off, a measured cost
table), simulate --gantt text, and sweep.  Run here, where /root/reference
exists:   python tests/golden/make_cli_golden.py

Each command runs the unmodified reference in a subprocess from a scratch
directory; the files it writes and its stdout/exit code go to cli.json.
tests/test_gpu_cli.py replays the same commands in-process with
paper_2103_16063_b200.install() (the device path behind the same CLI) and
compares byte for byte.
"""

import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"

CLUSTER = {"num_nodes": 2, "devices_per_node": 2, "device_memory_bytes": 4 * 2 ** 30,
           "bw_intra": 50e9, "bw_inter": 10e9, "link_latency_sec": 1e-5}
TABLE = {
    "matmul||mb=4": {"microbatch": 4, "t_fwd": 2.5e-4, "t_bwd": 6.0e-4},
    "matmul||mb=8": {"microbatch": 8, "t_fwd": 4.75e-4},
    "gelu||mb=8": {"microbatch": 8, "t_fwd": 3.0e-5, "act_bytes": 123456},
    "softmax||mb=4": {"microbatch": 4, "t_fwd": 1.5e-5, "t_bwd": 2.0e-5, "act_bytes": 4096},
    "add_layernorm||mb=2": {"microbatch": 2, "t_fwd": 9.0e-6},
    "matmul||mb=1": {"microbatch": 1, "t_fwd": 1.1e-5},
    "gelu||mb=1": {"microbatch": 1, "t_fwd": 4.0e-6, "act_bytes": 2048},
}
COMMON = ["--cluster", "cluster.json", "--batch-size", "32", "--k", "8"]
COMMANDS = [
    ("generate", ["generate", "bert", "--hidden", "256", "--layers", "4", "--seq", "64",
                  "--vocab", "1000", "--out", "g.json"]),
    ("partition", ["partition", "--graph", "g.json", *COMMON, "--oracle-check", "--out", "part"]),
    ("partition_nockpt", ["partition", "--graph", "g.json", *COMMON, "--checkpointing", "off",
                          "--out", "part_nock"]),
    ("partition_table", ["partition", "--graph", "g.json", *COMMON, "--cost-table", "table.json",
                         "--oracle-check", "--out", "part_ct"]),
    ("simulate", ["simulate", "--plan", "part/plan.json", "--graph", "g.json", *COMMON,
                  "--gantt", "text", "--out", "sim"]),
    ("sweep", ["sweep", "--cluster", "cluster.json", "--hidden", "128,256", "--layers", "2,3",
               "--seq", "64", "--vocab", "1000", "--batch-size", "32", "--k", "8",
               "--out", "sweep.csv"]),
]
OUTPUTS = ["part/plan.json", "part/blocks.json", "part/report.txt", "part_nock/plan.json",
           "part_nock/report.txt", "part_ct/plan.json", "part_ct/report.txt", "sim/gantt.txt",
           "sweep.csv"]


def setup(workdir):
    with open(os.path.join(workdir, "cluster.json"), "w") as fh:
        json.dump(CLUSTER, fh)
    with open(os.path.join(workdir, "table.json"), "w") as fh:
        json.dump(TABLE, fh)


def main():
    out = {"commands": [], "files": {}}
    with tempfile.TemporaryDirectory() as wd:
        setup(wd)
        env = dict(os.environ, PYTHONPATH=REF)
        for name, argv in COMMANDS:
            p = subprocess.run([sys.executable, "-c",
                                "import sys; from pipecut.cli import main; sys.exit(main(sys.argv[1:]))",
                                *argv], cwd=wd, env=env, capture_output=True, text=True)
            out["commands"].append({"name": name, "argv": argv, "rc": p.returncode,
                                    "stdout": p.stdout})
            print(name, p.returncode, p.stdout.strip().splitlines()[-1:], p.stderr[-300:])
        for f in OUTPUTS:
            with open(os.path.join(wd, f)) as fh:
                out["files"][f] = fh.read()
    with open(os.path.join(HERE, "cli.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")


def criterion8():
    """The acceptance gate's criterion-8 sweep (test_acceptance.py:324-353) with
    the reference CLI -> golden/sweep_c8.csv."""
    with tempfile.TemporaryDirectory() as wd:
        with open(os.path.join(wd, "cluster.json"), "w") as fh:
            json.dump({"num_nodes": 2, "devices_per_node": 2, "device_memory_bytes": 32 * 10 ** 9,
                       "bw_intra": 50e9, "bw_inter": 10e9, "link_latency_sec": 0.0}, fh)
        env = dict(os.environ, PYTHONPATH=REF)
        subprocess.run([sys.executable, "-c",
                        "import sys; from pipecut.cli import main; sys.exit(main(sys.argv[1:]))",
                        "sweep", "--cluster", "cluster.json", "--hidden", "2048",
                        "--layers", "24,48,96,192", "--batch-size", "32", "--out", "."],
                       cwd=wd, env=env, check=True)
        with open(os.path.join(wd, "sweep.csv")) as src, \
                open(os.path.join(HERE, "sweep_c8.csv"), "w") as dst:
            dst.write(src.read())


if __name__ == "__main__":
    main()
    if "c8" in sys.argv[1:]:
        criterion8()
