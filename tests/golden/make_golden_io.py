"""Golden point-cloud files written by the REFERENCE's own write_points
(pipeline_io.cpp, compiled by path into oracle/_ref). Run where
/root/reference exists:  python tests/golden/make_golden_io.py

Deliberately numpy-free: inside a process that has imported numpy, the
reference's ostream integer formatting in a ctypes-loaded library crashes
(observed here), so the points come from `random` and plain ctypes arrays.
"""
import ctypes as C
import json
import os
import random
import struct

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "libgeoshoot_ref.so")


def main():
    L = C.CDLL(REF)
    L.ref_write_points.argtypes = [C.c_char_p, C.c_int, C.c_int64, C.POINTER(C.c_double), C.c_char_p]
    rng = random.Random(3)
    vals = [rng.gauss(0, 1) * s for _ in range(101) for s in (1e-300, 1.0, 1e300)]
    vals[:3] = [0.1, -0.0, 5e-324]
    arr = (C.c_double * len(vals))(*vals)
    with open(os.path.join(HERE, "io_points.bin"), "wb") as f:
        f.write(struct.pack(f"<{len(vals)}d", *vals))
    for vtk, name in ((0, "io_ref.xyz"), (1, "io_ref.vtk")):
        st = L.ref_write_points(os.path.join(HERE, name).encode(), vtk, len(vals) // 3, arr, b"title")
        assert st == 0, st
    json.dump({"n": len(vals) // 3, "header": "title", "provenance": "reference write_points"},
              open(os.path.join(HERE, "io_ref.json"), "w"))
    print("wrote io_ref.xyz io_ref.vtk io_points.bin")


if __name__ == "__main__":
    main()
