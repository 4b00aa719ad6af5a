"""Checked build of libnbx.so: every source compiled with -DNBX_CHECKED=1 (device-side range
checks on list / grid / caller indices that print and trap on a violation; nbx_internal.cuh
NBX_DCHECK) into scratch/checked/libnbx.so.  Run the GPU tests against it with

    python tools/checked_build.py && NBX_LIB=scratch/checked/libnbx.so python -m pytest tests -m gpu

(the stand-in for compute-sanitizer memcheck, which this GPU pool does not run).
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "scratch", "checked")


def main():
    sys.path.insert(0, ROOT)
    from paper_2405_01420_b200 import build as B
    os.makedirs(OUT, exist_ok=True)
    cmds, objs = [], []
    for src in B.SOURCES:
        o = os.path.join(OUT, src.replace(".cu", ".o"))
        objs.append(o)
        cmds.append([B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, *B.PER_FILE.get(src, []), "-DNBX_CHECKED=1", "-c",
                     os.path.join(B.CSRC, src), "-o", o])
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        for c, r in zip(cmds, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds)):
            if r.returncode:
                sys.stderr.write(" ".join(c) + "\n" + r.stderr)
                raise SystemExit(1)
    lib = os.path.join(OUT, "libnbx.so")
    subprocess.check_call([B._nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart", "-lcufft"])
    print(lib)


if __name__ == "__main__":
    main()
