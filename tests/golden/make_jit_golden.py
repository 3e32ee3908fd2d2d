"""Regenerates tests/golden/jit_golden.json (and trace_t05.vptx): DSL kernels compiled by the
reference's own front end and run by its emulator (oracle/ref_jit_golden.cpp,
built from /root/reference by `make -C oracle _ref/jit_golden`)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/jit_golden"])
    out = subprocess.check_output([os.path.join(ROOT, "oracle", "_ref", "jit_golden")])
    with open(os.path.join(ROOT, "tests", "golden", "jit_golden.json"), "wb") as f:
        f.write(out)
    # the trace kernel's own VPTX (oracle/trace_t05.krn through the reference front end)
    vptx = subprocess.check_output([os.path.join(ROOT, "oracle", "_ref", "jit_golden"), "--trace-vptx",
                                    os.path.join(ROOT, "oracle", "trace_t05.krn")])
    with open(os.path.join(ROOT, "tests", "golden", "trace_t05.vptx"), "wb") as f:
        f.write(vptx)
