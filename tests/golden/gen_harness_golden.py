"""Golden fixtures for the config parser and the study harness, generated
from the UNMODIFIED reference (oracle/_ref via oracle/ref_lib.py; this
container only).  Re-run with  python tests/golden/gen_harness_golden.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref_lib as R  # noqa: E402

PARSE_CASES = [
    "",
    "# comment only\n\n",
    "order = 3\ncells_x = 4\ncells_y = 2 # trailing comment\nlength_x = 2.5\n",
    "jacobian_storage = initial-tuned\nfixed_faces = -x +y -z\ntraction_face = +x\ntraction_z = -0.02\n",
    "mu = 2.0\nlambda = 3.0\nsolver = lbfgs\nline_search = none\nload_steps = 4\n",
    "study_cases = 1x1 2x1 3x2\nstudy_reference = 4x4\nperf_orders = 2 4\nperf_target_dofs = 100 2000\n",
    "perf_representations = assembled\nperf_repeats = 7\ndeterministic = yes\nwrite_vtk = off\n",
    "body_force_x = 0.5\nbody_force_y = -1e-3\nmg_pre_smooth = 2\nmg_post_smooth = 3\n",
    "newton_rtol = 1e-6\nnewton_atol = 1e-9\nnewton_max_iterations = 12\nlinear_rtol = 1e-4\n"
    "linear_max_iterations = 99\nlbfgs_memory = 7\nprecond_refresh = 3\nthreads = 8\n",
    # errors
    "foo = 1\n",
    "order 3\n",
    "order = three\n",
    "cells_x = 2.5\n",
    "length_y = abc\n",
    "fixed_faces = -x +w\n",
    "traction_face = top\n",
    "jacobian_storage = fancy\n",
    "solver = gmres\n",
    "line_search = armijo\n",
    "deterministic = maybe\n",
    "study_cases = 2y2\n",
    "study_cases = 0x1\n",
    "perf_representations = dense\n",
    " = 4\n",
]

ACCURACY = """# small accuracy study with a body force and a traction
length_x = 2
cells_x = 2
traction_face = +x
traction_z = -0.02
body_force_z = -0.01
study_cases = 1x1 2x1 1x2
study_reference = 2x2
"""

PERFORMANCE = """perf_orders = 1 2 3
perf_target_dofs = 500 3000
perf_repeats = 3
"""


def main():
    parse = []
    for text in PARSE_CASES:
        try:
            parse.append({"text": text, "dump": R.parse_config(text)})
        except R.RefError as e:
            parse.append({"text": text, "error": str(e).split("] ", 1)[-1]})
    out = {"parse": parse, "accuracy_config": ACCURACY, "accuracy_csv": R.accuracy_study(ACCURACY),
           "performance_config": PERFORMANCE, "performance_csv": R.performance_study(PERFORMANCE)}
    with open(os.path.join(HERE, "harness.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("ok")


if __name__ == "__main__":
    main()
