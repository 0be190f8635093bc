"""Build the checked library (every translation unit with -DMS_CHECKS=1: bounds and
alignment checks in the kernels' memory movement, ms_common.cuh MS_CHECK) into
paper_2605_23727_b200/_variants/lib_checked.so. Run the GPU tests against it with
MS_LIB_PATH=<that file> (tools/gpu_checked.sh)."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import build as B  # noqa: E402


def main():
    out = B.PKG / "_variants"
    out.mkdir(exist_ok=True)
    nvcc = B._nvcc()

    def one(tu):
        obj = out / f"{tu}_checked.o"
        subprocess.run([nvcc, *B._host_cxx(), *B.NVCC_FLAGS, "-DMS_CHECKS=1", "-I", str(ROOT / "include"), "-c",
                        str(B.CSRC / tu), "-o", str(obj)], check=True)
        return str(obj)

    with ThreadPoolExecutor(len(B.SOURCES)) as ex:
        objs = list(ex.map(one, B.SOURCES))
    lib = out / "lib_checked.so"
    subprocess.run([nvcc, *B._host_cxx(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(lib),
                    *objs, "-lcudadevrt", "-lcuda"], check=True)
    print("built", lib)


if __name__ == "__main__":
    main()
