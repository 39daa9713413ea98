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


VTK_CASES = [(2, (2, 1, 1), (2.0, 1.0, 1.0)), (3, (1, 2, 1), (1.0, 1.5, 0.7)),
             (1, (2, 2, 2), (1.0, 1.0, 1.0))]

# The reference's write_vtk formats doubles through std::ostream, which
# crashes once numpy's bundled libraries are in the process; run it in a
# ctypes-only child.
_VTK_CHILD = r"""
import ctypes, json, math, sys
order, cells, ext = json.loads(sys.argv[1])
L = ctypes.CDLL(sys.argv[2])
L.ref_create.restype = ctypes.c_void_p
h = L.ref_create((ctypes.c_double * 3)(*ext), (ctypes.c_int * 3)(*cells), order, 0, 1, -1,
                 (ctypes.c_double * 3)(0, 0, 0), ctypes.c_double(1.0), ctypes.c_double(0.3), 1)
n = L.ref_size(ctypes.c_void_p(h))
u = (ctypes.c_double * n)(*[1.2345678912345e-3 * math.sin(0.37 * i) for i in range(n)])
buf = ctypes.create_string_buffer(1 << 22)
assert L.ref_write_vtk(ctypes.c_void_p(h), u, buf, 1 << 22) == 0
sys.stdout.write(buf.value.decode())
"""


def gen_vtk():
    import subprocess
    out = []
    for order, cells, ext in VTK_CASES:
        text = subprocess.run([sys.executable, "-c", _VTK_CHILD, json.dumps([order, cells, ext]),
                               R.LIB_PATH], check=True, capture_output=True, text=True).stdout
        out.append({"order": order, "cells": cells, "extents": ext, "vtk": text})
    return out


def main():
    parse = []
    for text in PARSE_CASES:
        try:
            parse.append({"text": text, "dump": R.parse_config(text)})
        except R.RefError as e:
            parse.append({"text": text, "error": str(e).split("] ", 1)[-1]})
    out = {"parse": parse, "accuracy_config": ACCURACY, "accuracy_csv": R.accuracy_study(ACCURACY),
           "performance_config": PERFORMANCE, "performance_csv": R.performance_study(PERFORMANCE),
           "vtk": gen_vtk()}
    with open(os.path.join(HERE, "harness.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("ok")


if __name__ == "__main__":
    main()
