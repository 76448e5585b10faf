"""Record the REAL reference CLI's reports as golden fixtures for tests/test_cli.py.

Run in the build container (the reference is installed into oracle/_ref by
oracle/build_ref.sh):

    python tests/golden/make_cli_golden.py

Every case runs `python -m gemap <args>` from the reference build with its
working directory at tests/golden/cli/, so the relative paths echoed in the
manifests are the ones the test uses. The input trace/profile files are
themselves written by the reference (gen-trace / gen-profile) and committed
under tests/golden/cli/inputs/. Outputs (stdout, plus any files a command
writes) go to tests/golden/cli/expected/<case>/.
"""

from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = ROOT / "oracle" / "_ref"
CLI = HERE / "cli"

# (case, args, files the command writes relative to the cwd)
INPUTS = [
    ("trace_a", ["gen-trace", "--experts", "8", "--steps", "24", "--tokens-per-step", "256", "--consistent", "0,3",
                 "--temporal", "1,5:0.3:3", "--seed", "11", "--output", "inputs/trace_a.json", "--quiet"]),
    ("trace_b", ["gen-trace", "--experts", "8", "--steps", "16", "--seed", "12", "--format", "csv",
                 "--output", "inputs/trace_b.csv", "--quiet"]),
    ("layer0", ["gen-trace", "--experts", "16", "--steps", "20", "--consistent", "2", "--seed", "21",
                "--output", "inputs/layers/layer0.json", "--quiet"]),
    ("layer1", ["gen-trace", "--experts", "16", "--steps", "20", "--temporal", "3,4", "--seed", "22",
                "--output", "inputs/layers/layer1.json", "--quiet"]),
    ("layer2", ["gen-trace", "--experts", "16", "--steps", "20", "--seed", "23", "--format", "csv",
                "--output", "inputs/layers/layer2.csv", "--quiet"]),
    ("mixed0", ["gen-trace", "--experts", "16", "--steps", "20", "--seed", "31",
                "--output", "inputs/mixed/m0.json", "--quiet"]),
    ("mixed1", ["gen-trace", "--experts", "16", "--steps", "19", "--temporal", "1,2", "--seed", "32",
                "--output", "inputs/mixed/m1.json", "--quiet"]),
    ("mixed2", ["gen-trace", "--experts", "8", "--steps", "20", "--seed", "33", "--format", "csv",
                "--output", "inputs/mixed/m2.csv", "--quiet"]),
    ("profile4", ["gen-profile", "--gpus", "4", "--setup", "moderate", "--seed", "5", "--max-tokens", "2048",
                  "--output", "inputs/profile4.json", "--quiet"]),
    ("profile2", ["gen-profile", "--gpus", "2", "--setup", "high", "--tile", "32", "--max-tokens", "1024",
                  "--overhead", "0.25", "--output", "inputs/profile2.json", "--quiet"]),
    ("linear_a", ["baseline", "linear", "--trace", "inputs/trace_a.json", "--gpus", "4",
                  "--output", "inputs/linear_a.json", "--quiet"]),
    ("eplb_a", ["baseline", "eplb", "--trace", "inputs/trace_a.json", "--gpus", "4",
                "--output", "inputs/eplb_a.json", "--quiet"]),
]

CASES = [
    ("gen_trace_stdout", ["gen-trace", "--experts", "6", "--steps", "5", "--tokens-per-step", "64", "--seed", "3",
                          "--quiet"], []),
    ("gen_trace_csv_stdout", ["gen-trace", "--experts", "4", "--steps", "3", "--seed", "4", "--format", "csv",
                              "--quiet"], []),
    ("gen_profile_stdout", ["gen-profile", "--gpus", "3", "--setup", "explicit", "--speed-factors", "1,0.9,1.2",
                            "--max-tokens", "512", "--quiet"], []),
    ("baseline_linear_stdout", ["baseline", "linear", "--trace", "inputs/trace_b.csv", "--gpus", "2", "--quiet"], []),
    ("baseline_eplb_stdout", ["baseline", "eplb", "--trace", "inputs/trace_a.json", "--gpus", "4", "--quiet"], []),
    ("stats_a", ["stats", "--trace", "inputs/trace_a.json"], []),
    ("stats_b", ["stats", "--trace", "inputs/trace_b.csv"], []),
    ("score_a", ["score", "--trace", "inputs/trace_a.json", "--profile", "inputs/profile4.json",
                 "--mapping", "inputs/eplb_a.json"], []),
    ("replay_a", ["replay", "--trace", "inputs/trace_a.json", "--profile", "inputs/profile4.json",
                  "--mapping", "inputs/linear_a.json"], []),
    ("compare_a", ["compare", "--trace", "inputs/trace_a.json", "--profile", "inputs/profile4.json",
                   "inputs/linear_a.json", "inputs/eplb_a.json"], []),
    ("optimize_a", ["optimize", "--trace", "inputs/trace_a.json", "--profile", "inputs/profile4.json",
                    "--seed", "7", "--restarts", "6", "--mapping-out", "out/best_a.json"], ["out/best_a.json"]),
    ("optimize_b", ["optimize", "--trace", "inputs/trace_b.csv", "--profile", "inputs/profile2.json",
                    "--seed", "9", "--no-baseline-seeds", "--restarts", "4"], []),
    ("multi_layer", ["multi-layer", "--trace-dir", "inputs/layers", "--profile", "inputs/profile4.json",
                     "--output-dir", "out/ml", "--seed", "13", "--restarts", "5"],
     ["out/ml/layer0.mapping.json", "out/ml/layer1.mapping.json", "out/ml/layer2.mapping.json"]),
    ("multi_layer_mixed", ["multi-layer", "--trace-dir", "inputs/mixed", "--profile", "inputs/profile4.json",
                           "--output-dir", "out/mx", "--seed", "17", "--restarts", "4"],
     ["out/mx/m0.mapping.json", "out/mx/m1.mapping.json", "out/mx/m2.mapping.json"]),
    ("bad_gpus", ["baseline", "linear", "--trace", "inputs/trace_a.json", "--gpus", "3"], []),
    ("missing_trace", ["stats", "--trace", "inputs/nope.json"], []),
]


def run_ref(args, cwd):
    env = dict(os.environ, PYTHONPATH=str(REF), GEM_BACKEND="cython")
    return subprocess.run([sys.executable, "-m", "gemap", *args], cwd=cwd, env=env, capture_output=True, text=True)


def main() -> None:
    assert (REF / "gemap").is_dir(), "build the reference first: bash oracle/build_ref.sh"
    shutil.rmtree(CLI, ignore_errors=True)
    (CLI / "inputs" / "layers").mkdir(parents=True)
    (CLI / "inputs" / "mixed").mkdir(parents=True)
    for name, args in INPUTS:
        p = run_ref(args, CLI)
        assert p.returncode == 0, (name, p.stderr)
    index = []
    for name, args, files in CASES:
        shutil.rmtree(CLI / "out", ignore_errors=True)
        (CLI / "out").mkdir()
        p = run_ref(args, CLI)
        dest = CLI / "expected" / name
        dest.mkdir(parents=True)
        (dest / "stdout").write_text(p.stdout)
        for f in files:
            shutil.copy(CLI / f, dest / Path(f).name)
        index.append({"case": name, "args": args, "returncode": p.returncode, "files": files})
    shutil.rmtree(CLI / "out", ignore_errors=True)
    (CLI / "cases.json").write_text(json.dumps(index, indent=1) + "\n")
    print(f"wrote {len(index)} CLI cases under {CLI}")


if __name__ == "__main__":
    main()
