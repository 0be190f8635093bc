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
    "g1": {},
    "g2": {"MS_TMA_KB_F64": 65536, "MS_TMA_RPW_F64": 2, "MS_TMA_KB_K16": 49152},
    "g3": {"MS_TMA_KB_F64": 32768, "MS_TMA_KB_K16": 24576},
    "g4": {"MS_TMA_KB_F32": 49152, "MS_TMA_KB_K16": 65536},
    "g5": {"MS_TMA_KB_F32": 81920, "MS_TMA_KB_K16": 16384},
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
        others = [str(B.BUILD / (src + ".o")) for src in B.SOURCES if src != "ms_rhs_fast.cu"]
        subprocess.run([nvcc, *B._host_cxx(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(lib),
                        *others, str(obj), "-lcudadevrt"], check=True)
        return name

    items = [(k, v) for k, v in VARIANTS.items() if not names or k in names]
    with ThreadPoolExecutor(8) as ex:
        for n in ex.map(one, items):
            print("built", n)


if __name__ == "__main__":
    main(sys.argv[1:])
