"""Build geometry variants of the K-sweep kernel (same sources, -D overrides of
MS_FAST_THREADS / MS_FAST_MINB / MS_FAST_R / MS_CHUNK / MS_NS / MS_PREFETCH)
into paper_2605_23727_b200/_variants/lib_<name>.so for tools/tune_rhs.py."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2605_23727_b200 import build as B  # noqa: E402

VARIANTS = {
    "base": {},
    "r4": {"MS_FAST_R": 4},
    "t256x2": {"MS_FAST_THREADS": 256, "MS_FAST_MINB": 2},
    "t1024r4": {"MS_FAST_THREADS": 1024, "MS_FAST_R": 4},
    "c2048": {"MS_CHUNK": 2048},
    "c1024": {"MS_CHUNK": 1024},
    "c4096ns3": {"MS_CHUNK": 4096, "MS_NS": 3},
    "pfr4": {"MS_PREFETCH": 1, "MS_FAST_R": 4},
    "pfr6": {"MS_PREFETCH": 1, "MS_FAST_R": 6},
    "pfr4t256x2": {"MS_PREFETCH": 1, "MS_FAST_R": 4, "MS_FAST_THREADS": 256, "MS_FAST_MINB": 2},
}


def main(names=None):
    B.build_library()
    out = B.PKG / "_variants"
    out.mkdir(exist_ok=True)
    nvcc = B._nvcc()

    def one(item):
        name, defs = item
        obj = out / f"rhs_fast_{name}.o"
        lib = out / f"lib_{name}.so"
        dflags = [f"-D{k}={v}" for k, v in defs.items()]
        subprocess.run([nvcc, *B._host_cxx(), *B.NVCC_FLAGS, *dflags, "-I", str(ROOT / "include"), "-c",
                        str(B.CSRC / "ms_rhs_fast.cu"), "-o", str(obj)], check=True)
        subprocess.run([nvcc, *B._host_cxx(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(lib),
                        str(B.BUILD / "ms_api.cu.o"), str(obj), str(B.BUILD / "ms_rhs_faithful.cu.o"), "-lcudadevrt"],
                       check=True)
        return name

    items = [(k, v) for k, v in VARIANTS.items() if not names or k in names]
    with ThreadPoolExecutor(8) as ex:
        for n in ex.map(one, items):
            print("built", n)


if __name__ == "__main__":
    main(sys.argv[1:])
