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

# name -> (translation unit to rebuild, -D overrides)
VARIANTS = {
    "tc_base": ("ms_batch.cu", {}),
    "tc_s2x2": ("ms_batch.cu", {"MS_TC_STAGES": 2, "MS_TC_MINB": 2}),
    "tc_e8": ("ms_batch.cu", {"MS_TC_EPI_WARPS": 8}),
    "tc_s2x2_e8": ("ms_batch.cu", {"MS_TC_STAGES": 2, "MS_TC_MINB": 2, "MS_TC_EPI_WARPS": 8}),
    "tc_s3_e8": ("ms_batch.cu", {"MS_TC_STAGES": 3, "MS_TC_EPI_WARPS": 8}),
    # CTA-pair kernel: tile width, ring depth, CTAs per SM, epilogue off (mainloop time)
    "tc2_n512_s4": ("ms_batch.cu", {}),
    "tc2_n512_s4_noepi": ("ms_batch.cu", {"MS_T2_NOEPI": 1}),
    "tc2_packed": ("ms_batch.cu", {"MS_TC_PACKED": 1}),
    "tc2_split": ("ms_batch.cu", {"MS_TC_PACKED": 0}),
    "tc2_n512_s3": ("ms_batch.cu", {"MS_T2_STAGES": 3}),
    "tc2_n256_s4": ("ms_batch.cu", {"MS_T2_BN": 256, "MS_T2_STAGES": 4}),
    "tc2_n256_s3x2": ("ms_batch.cu", {"MS_T2_BN": 256, "MS_T2_STAGES": 3, "MS_T2_MINB": 2}),
    "tc2_n256_s2x2": ("ms_batch.cu", {"MS_T2_BN": 256, "MS_T2_STAGES": 2, "MS_T2_MINB": 2}),
    "tc2_n512_s4_e16": ("ms_batch.cu", {"MS_T2_EPI": 16}),
    "tc2_n512_s3_e16": ("ms_batch.cu", {"MS_T2_EPI": 16, "MS_T2_STAGES": 3}),
    "tc2_n256_s3x2_e16": ("ms_batch.cu", {"MS_T2_BN": 256, "MS_T2_STAGES": 3, "MS_T2_MINB": 2, "MS_T2_EPI": 16}),
    # fused small-system evaluation: rows per warp x column-loop unroll
    "fused_r2u4": ("ms_rhs_fast.cu", {}),
    "fused_r1u8": ("ms_rhs_fast.cu", {"MS_FUSED_R": 1, "MS_FUSED_UNROLL": 8}),
    "fused_r2u8": ("ms_rhs_fast.cu", {"MS_FUSED_R": 2, "MS_FUSED_UNROLL": 8}),
    "fused_r4u2": ("ms_rhs_fast.cu", {"MS_FUSED_R": 4, "MS_FUSED_UNROLL": 2}),
    "fused_r8u1": ("ms_rhs_fast.cu", {"MS_FUSED_R": 8, "MS_FUSED_UNROLL": 1}),
    "fused_r1u16": ("ms_rhs_fast.cu", {"MS_FUSED_R": 1, "MS_FUSED_UNROLL": 16}),
    "fused_r1u4": ("ms_rhs_fast.cu", {"MS_FUSED_R": 1, "MS_FUSED_UNROLL": 4}),
    # concurrent-variant sweep (ms_multi.cuh): consumer warps x rows per warp
    "multi_w8r4": ("ms_multi.cu", {}),
    "multi_w16r2": ("ms_multi.cu", {"MS_MULTI_WARPS": 16, "MS_MULTI_R": 2}),
    "multi_w12r4": ("ms_multi.cu", {"MS_MULTI_WARPS": 12, "MS_MULTI_R": 4}),
    "multi_w8r2": ("ms_multi.cu", {"MS_MULTI_WARPS": 8, "MS_MULTI_R": 2}),
    "multi_w16r2_i": ("ms_multi.cu", {"MS_MULTI_WARPS": 16, "MS_MULTI_R": 2, "MS_MULTI_INTCVT": 1}),
    "multi_w12r2": ("ms_multi.cu", {"MS_MULTI_WARPS": 12, "MS_MULTI_R": 2}),
    "multi_w16r3": ("ms_multi.cu", {"MS_MULTI_WARPS": 16, "MS_MULTI_R": 3}),
    "multi_w20r2": ("ms_multi.cu", {"MS_MULTI_WARPS": 20, "MS_MULTI_R": 2}),
    "multi_w16r4": ("ms_multi.cu", {"MS_MULTI_WARPS": 16, "MS_MULTI_R": 4}),
    "multi_w24r2": ("ms_multi.cu", {"MS_MULTI_WARPS": 24, "MS_MULTI_R": 2}),
    # cp.async.bulk K sweep with 16-bit K: rows per consumer warp x K bytes per stage
    "base": ("ms_rhs_fast.cu", {}),
    "t16_r2_32k": ("ms_rhs_fast.cu", {"MS_TMA_RPW_K16": 2}),
    "t16_r4_32k": ("ms_rhs_fast.cu", {"MS_TMA_RPW_K16": 4}),
    "t16_r2_64k": ("ms_rhs_fast.cu", {"MS_TMA_RPW_K16": 2, "MS_TMA_KB_K16": 65536}),
    "t16_r4_64k": ("ms_rhs_fast.cu", {"MS_TMA_RPW_K16": 4, "MS_TMA_KB_K16": 65536}),
    "t16_r1_64k": ("ms_rhs_fast.cu", {"MS_TMA_KB_K16": 65536}),
    # TMA f32 sweep in the power-capped (sustained) regime, tools/sustained_sweep.py
    "tf_r2": ("ms_rhs_fast.cu", {"MS_TMA_RPW_F32": 2}),
    "tf_c8r2": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 8, "MS_TMA_RPW_F32": 2}),
    "tf_c8": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 8}),
    "tf_32k_s6": ("ms_rhs_fast.cu", {"MS_TMA_KB_F32": 32768, "MS_TMA_STAGES": 6}),
    "tf_c8_32k_s6": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 8, "MS_TMA_KB_F32": 32768, "MS_TMA_STAGES": 6}),
    "tf_c4r4": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 4, "MS_TMA_RPW_F32": 4}),
    "tf_c8r2_48k": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 8, "MS_TMA_RPW_F32": 2, "MS_TMA_KB_F32": 49152}),
    "tf_c8r4": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 8, "MS_TMA_RPW_F32": 4}),
    "tf_c4r8": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 4, "MS_TMA_RPW_F32": 8}),
    "tf_c8r2_1l": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 8, "MS_TMA_RPW_F32": 2, "MS_TMA_LANES": 0}),
    "tf_c8r2d4": ("ms_rhs_fast.cu", {"MS_TMA_CONS": 8, "MS_TMA_RPW_F32": 2, "MS_TMA_RPW_F64": 4}),
    "tf_sss_c16r1": ("ms_rhs_fast.cu", {"MS_TMA_CONS_SSS": 16, "MS_TMA_RPW_SSS": 1}),
    "tf_khint": ("ms_rhs_fast.cu", {"MS_TMA_KHINT": 1}),
    "hint_off": ("ms_rhs_fast.cu", {"MS_TMA_KHINT": 0, "MS_LDG_KHINT": 0}),
    "multi_nohint": ("ms_multi.cu", {"MS_MULTI_KHINT": 0}),
    "prep_e2": ("ms_batch.cu", {"MS_PREP_TC_ELEMS": 2}),
    "prep_e4": ("ms_batch.cu", {"MS_PREP_TC_ELEMS": 4}),
    "prep_e8": ("ms_batch.cu", {"MS_PREP_TC_ELEMS": 8}),
    "fin_m4": ("ms_batch.cu", {"MS_BFIN_MINB": 1}),
    "fin_m6": ("ms_batch.cu", {"MS_BFIN_MINB": 6}),
    "fin_m8": ("ms_batch.cu", {"MS_BFIN_MINB": 8}),
    "tc2_n256_s3x2_noepi": ("ms_batch.cu", {"MS_T2_BN": 256, "MS_T2_STAGES": 3, "MS_T2_MINB": 2, "MS_T2_NOEPI": 1}),
    # packed FADD2 accumulation (ms_common.cuh add2) and the 16-bit K TMA sweep geometry
    "nofadd2": ("ms_rhs_fast.cu", {"MS_NO_FADD2": 1}),
    "k16_c8r2": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 8, "MS_TMA_RPW_K16": 2}),
    "k16_c8r2_64k": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 8, "MS_TMA_RPW_K16": 2, "MS_TMA_KB_K16": 65536}),
    "k16_c8r2_64k_nofadd2": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 8, "MS_TMA_RPW_K16": 2, "MS_TMA_KB_K16": 65536,
                                                "MS_NO_FADD2": 1}),
    "k16_c8r4_64k": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 8, "MS_TMA_RPW_K16": 4, "MS_TMA_KB_K16": 65536}),
    "k16_c16r2_64k": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 16, "MS_TMA_RPW_K16": 2, "MS_TMA_KB_K16": 65536}),
    "k16_c4r4_64k": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 4, "MS_TMA_RPW_K16": 4, "MS_TMA_KB_K16": 65536}),
    "u1": ("ms_rhs_fast.cu", {"MS_TMA_UNROLL": 1}),
    "u2": ("ms_rhs_fast.cu", {"MS_TMA_UNROLL": 2}),
    "u8": ("ms_rhs_fast.cu", {"MS_TMA_UNROLL": 8}),
    "k16_c16r2_64k_u2": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 16, "MS_TMA_RPW_K16": 2, "MS_TMA_KB_K16": 65536,
                                            "MS_TMA_UNROLL": 2}),
    "k16_c16r2_64k_nofadd2": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 16, "MS_TMA_RPW_K16": 2, "MS_TMA_KB_K16": 65536,
                                                 "MS_NO_FADD2": 1}),
    "k16_c8r8_64k": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 8, "MS_TMA_RPW_K16": 8}),
    "k16_c4r8_64k": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 4, "MS_TMA_RPW_K16": 8}),
    "k16_c8r4_48k": ("ms_rhs_fast.cu", {"MS_TMA_KB_K16": 49152}),
    "k16_c8r4_32k_s6": ("ms_rhs_fast.cu", {"MS_TMA_KB_K16": 32768, "MS_TMA_STAGES": 6}),
    "k16_c8r4_u1": ("ms_rhs_fast.cu", {"MS_TMA_UNROLL": 1}),
    "k16_c8r4_u2": ("ms_rhs_fast.cu", {"MS_TMA_UNROLL": 2}),
    "fin_small4k": ("ms_api.cu", {"MS_FIN_SMALL_MAX": 4096}),
    "fin_small8k": ("ms_api.cu", {"MS_FIN_SMALL_MAX": 8192}),
    "tf_sss_c16r1_32k_s6": ("ms_rhs_fast.cu", {"MS_TMA_CONS_SSS": 16, "MS_TMA_RPW_SSS": 1, "MS_TMA_KB_F32": 32768,
                                               "MS_TMA_STAGES": 6}),
    "tf_sss_32k_s6": ("ms_rhs_fast.cu", {"MS_TMA_KB_F32": 32768, "MS_TMA_STAGES": 6}),
    "tf_sss_16k_s8": ("ms_rhs_fast.cu", {"MS_TMA_KB_F32": 16384, "MS_TMA_STAGES": 8}),
    "tma_m2_32k_s3": ("ms_rhs_fast.cu", {"MS_TMA_MINB": 2, "MS_TMA_KB_F32": 32768, "MS_TMA_STAGES": 3}),
    "tma_m2_48k_s2": ("ms_rhs_fast.cu", {"MS_TMA_MINB": 2, "MS_TMA_KB_F32": 49152, "MS_TMA_STAGES": 2}),
    "tma_m2_24k_s4": ("ms_rhs_fast.cu", {"MS_TMA_MINB": 2, "MS_TMA_KB_F32": 24576, "MS_TMA_STAGES": 4}),
    "tc_rec1": ("ms_batch.cu", {"MS_TC_PACKED": 1}),
    "fast_fadd2": ("ms_rhs_fast.cu", {"MS_FAST_FADD2": 1}),
    "fin_t128_u4": ("ms_batch.cu", {"MS_BFIN_THREADS": 128, "MS_BFIN_UNROLL": 4}),
    "fin_t128_u8": ("ms_batch.cu", {"MS_BFIN_THREADS": 128, "MS_BFIN_UNROLL": 8}),
    "fin_t128": ("ms_batch.cu", {"MS_BFIN_THREADS": 128}),
    "fin_t256_u4": ("ms_batch.cu", {"MS_BFIN_UNROLL": 4}),
    "pow_libm_api": ("ms_api.cu", {"MS_POW_ROOT_START": 0}),
    "pow_libm_batch": ("ms_batch.cu", {"MS_POW_ROOT_START": 0}),
    "k16_c12r2_48k": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 12, "MS_TMA_RPW_K16": 2, "MS_TMA_KB_K16": 49152}),
    # round 2, packed FMUL2.FTZ products: register sweep rows per warp, 16-bit K TMA geometry
    "fr4": ("ms_rhs_fast.cu", {"MS_FAST_R": 4}),
    "fr12": ("ms_rhs_fast.cu", {"MS_FAST_R": 12}),
    "fr16": ("ms_rhs_fast.cu", {"MS_FAST_R": 16}),
    "fr8_t256": ("ms_rhs_fast.cu", {"MS_FAST_THREADS": 256, "MS_FAST_MINB": 2}),
    "pk_c16r2": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 16, "MS_TMA_RPW_K16": 2}),
    "pk_c8r2": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 8, "MS_TMA_RPW_K16": 2}),
    "pk_c4r8": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 4, "MS_TMA_RPW_K16": 8}),
    "pk_c8r8": ("ms_rhs_fast.cu", {"MS_TMA_CONS_K16": 8, "MS_TMA_RPW_K16": 8}),
    "pk_c8r4_32k_s6": ("ms_rhs_fast.cu", {"MS_TMA_KB_K16": 32768, "MS_TMA_STAGES": 6}),
    "pk_sss_c4r4": ("ms_rhs_fast.cu", {"MS_TMA_CONS_SSS": 4, "MS_TMA_RPW_SSS": 4}),
    "pk_sss_c4r2": ("ms_rhs_fast.cu", {"MS_TMA_CONS_SSS": 4, "MS_TMA_RPW_SSS": 2}),
    "f32_nopk": ("ms_rhs_fast.cu", {"MS_SWEEP_PK": 0}),
    "f32_pk_u2": ("ms_rhs_fast.cu", {"MS_TMA_UNROLL": 2}),
    "f32_pk_u8": ("ms_rhs_fast.cu", {"MS_TMA_UNROLL": 8}),
    "f32_pk_c16r1": ("ms_rhs_fast.cu", {"MS_TMA_CONS_SSS": 16, "MS_TMA_RPW_SSS": 1}),
    "f32_pk_c8r4": ("ms_rhs_fast.cu", {"MS_TMA_CONS_SSS": 8, "MS_TMA_RPW_SSS": 4}),
    "f32_pk_s3": ("ms_rhs_fast.cu", {"MS_TMA_STAGES": 3}),
    "tcx_halfb": ("ms_batch.cu", {"MS_T2_NOEPI": 1, "MS_T2_EXP_NB": 1}),
    "tcx_nob": ("ms_batch.cu", {"MS_T2_NOEPI": 1, "MS_T2_EXP_NB": 0}),
    "tcx_1mma": ("ms_batch.cu", {"MS_T2_NOEPI": 1, "MS_T2_EXP_NMMA": 1}),
    "tcx_0mma": ("ms_batch.cu", {"MS_T2_NOEPI": 1, "MS_T2_EXP_NMMA": 0}),
    "tcv_base": ("ms_batch.cu", {}),
    "tcv_rec64": ("ms_batch.cu", {"MS_TC_REC128": 0}),
    "tcv_stcg": ("ms_batch.cu", {"MS_TC_STCG": 1}),
    "tcv_fin": ("ms_batch.cu", {"MS_TC_FIN": 1}),
    "tcv_noepi": ("ms_batch.cu", {"MS_T2_NOEPI": 1}),
    # round 2: epilogue records staged in shared memory (default) vs per-thread loads
    "tcs_new": ("ms_batch.cu", {}),
    # C5 windowed accumulation (MS_T2_DRAIN k-blocks per window; 0 = one accumulator over all of K)
    "dr4": ("ms_batch.cu", {}),
    "dr2": ("ms_batch.cu", {"MS_T2_DRAIN": 2}),
    "dr8": ("ms_batch.cu", {"MS_T2_DRAIN": 8}),
    "dr3": ("ms_batch.cu", {"MS_T2_DRAIN": 3}),
    "dr2x8": ("ms_batch.cu", {"MS_T2_DRAIN": 2, "MS_T2_XWARPS": 8}),
    "dr3x8": ("ms_batch.cu", {"MS_T2_DRAIN": 3, "MS_T2_XWARPS": 8}),
    "dr0": ("ms_batch.cu", {"MS_T2_DRAIN": 0}),
    "drx_noadd": ("ms_batch.cu", {"MS_T2_EXP_DRAIN": 1}),
    "rege1": ("ms_batch.cu", {}),
    "rege0": ("ms_batch.cu", {"MS_T2_REGEPI": 0}),
    # C4 f32 TMA sweep: the first rows of every CTA's range kept in L2 (evict-last) across evaluations
    # f16 tensor-core sweep (MS_SWEEP=tc16): accumulator batch, TMEM groups, ring depth, no-TMEM-load timing
    "gv_kb4": ("ms_rhs_fast.cu", {}),
    "gv_cur": ("ms_rhs_fast.cu", {}),
    "gv_exp1": ("ms_rhs_fast.cu", {"MS_GV_EXP": 1}),
    "gv_g4": ("ms_rhs_fast.cu", {"MS_GV_GROUPS": 4}),
    "gv_fine1": ("ms_rhs_fast.cu", {}),
    "gv_fine0": ("ms_rhs_fast.cu", {"MS_GV_FINE": 0}),
    "gv_pf0": ("ms_rhs_fast.cu", {"MS_GV_PF": 0}),
    "gv_pf2": ("ms_rhs_fast.cu", {"MS_GV_PF": 2}),
    "gv_pf4": ("ms_rhs_fast.cu", {"MS_GV_PF": 4}),
    "gv_pf8": ("ms_rhs_fast.cu", {"MS_GV_PF": 8}),
    "gv_kb2": ("ms_rhs_fast.cu", {"MS_GV_KB": 2}),
    "gv_kb1": ("ms_rhs_fast.cu", {"MS_GV_KB": 1}),
    "gv_kb4_g4": ("ms_rhs_fast.cu", {"MS_GV_GROUPS": 4}),
    "gv_kb4_exp1": ("ms_rhs_fast.cu", {"MS_GV_EXP": 1}),
    "gv_fine_i1": ("ms_rhs_fast.cu", {"MS_GV_FINE": 1, "MS_GV_ISSUE": 1}),
    "gv_fine_i2": ("ms_rhs_fast.cu", {"MS_GV_FINE": 1, "MS_GV_ISSUE": 2}),
    "gv_fine_i4": ("ms_rhs_fast.cu", {"MS_GV_FINE": 1, "MS_GV_ISSUE": 4}),
    "gv_zatom": ("ms_rhs_fast.cu", {"MS_GV_ZATOM": 1}),
    "gv_rev0": ("ms_rhs_fast.cu", {"MS_GV_REV": 0}),
    "gv_rev1": ("ms_rhs_fast.cu", {"MS_GV_REV": 1}),
    "gv_keep32n": ("ms_rhs_fast.cu", {"MS_GV_KEEPKB": 32, "MS_GV_KEEPPOL": 1}),
    "gv_keep16n": ("ms_rhs_fast.cu", {"MS_GV_KEEPKB": 16, "MS_GV_KEEPPOL": 1}),
    "gv_keep32l": ("ms_rhs_fast.cu", {"MS_GV_KEEPKB": 32, "MS_GV_KEEPPOL": 2}),
    "gv_keep16l": ("ms_rhs_fast.cu", {"MS_GV_KEEPKB": 16, "MS_GV_KEEPPOL": 2}),
    "gv_fine_s12": ("ms_rhs_fast.cu", {"MS_GV_FINE": 1, "MS_GV_ISSUE": 1, "MS_GV_STAGES": 12}),
    "gv_fine_s8": ("ms_rhs_fast.cu", {"MS_GV_FINE": 1, "MS_GV_ISSUE": 1, "MS_GV_STAGES": 8}),
    "gv_kb2_s6z": ("ms_rhs_fast.cu", {"MS_GV_KB": 2, "MS_GV_STAGES": 6, "MS_GV_ZATOM": 1}),
    # round 2, fourth session: warp-uniform MMA issuer, prologue before griddepcontrol.wait, batched combine
    "gv_old": ("ms_rhs_fast.cu", {"MS_GV_UISSUE": 0, "MS_GV_PRE": 0, "MS_GV_COMB": 0}),
    "gv_u": ("ms_rhs_fast.cu", {"MS_GV_UISSUE": 1, "MS_GV_PRE": 0, "MS_GV_COMB": 0}),
    "gv_uc": ("ms_rhs_fast.cu", {"MS_GV_UISSUE": 1, "MS_GV_PRE": 0, "MS_GV_COMB": 1}),
    "gv_new": ("ms_rhs_fast.cu", {}),
    "gv_new_fine": ("ms_rhs_fast.cu", {"MS_GV_FINE": 1}),
    "gv_new_fine_i1": ("ms_rhs_fast.cu", {"MS_GV_FINE": 1, "MS_GV_ISSUE": 1}),
    "gv_new_kb2": ("ms_rhs_fast.cu", {"MS_GV_KB": 2, "MS_GV_STAGES": 6, "MS_GV_ZATOM": 1}),
    "gv_new_zatom": ("ms_rhs_fast.cu", {"MS_GV_ZATOM": 1}),
    "fin_u4": ("ms_api.cu", {"MS_FIN_UNROLL": 4}),
    "fin_u1": ("ms_api.cu", {"MS_FIN_UNROLL": 1}),
    "pow_cold0": ("ms_api.cu", {"MS_POW_COLD": 0}),
    "pow_cold1": ("ms_api.cu", {"MS_POW_COLD": 1}),
    "t2_pro0": ("ms_batch.cu", {"MS_T2_PRO_RELAXED": 0}),
    "t2_pro1": ("ms_batch.cu", {"MS_T2_PRO_RELAXED": 1}),
    "t2_rel0": ("ms_batch.cu", {"MS_T2_DRAIN_RELAXED": 0}),
    "t2_rel1": ("ms_batch.cu", {"MS_T2_DRAIN_RELAXED": 1}),
    "gv_ar0": ("ms_rhs_fast.cu", {"MS_GV_ATOMREL": 0}),
    "gv_ar1": ("ms_rhs_fast.cu", {"MS_GV_ATOMREL": 1}),
    "gv_ar1_own1": ("ms_rhs_fast.cu", {"MS_GV_ATOMREL": 1, "MS_GV_OWN": 1}),
    "gv_own0": ("ms_rhs_fast.cu", {"MS_GV_OWN": 0}),
    "gv_own1": ("ms_rhs_fast.cu", {"MS_GV_OWN": 1}),
    "gv_kbfull": ("ms_rhs_fast.cu", {"MS_GV_KBFULL": 1}),
    "gv_kbfull_z": ("ms_rhs_fast.cu", {"MS_GV_KBFULL": 1, "MS_GV_ZATOM": 1}),
    "gv_g8b2": ("ms_rhs_fast.cu", {"MS_GV_BATCH": 2}),
    "keep0": ("ms_rhs_fast.cu", {"MS_TMA_KEEP": 0}),
    "keep2": ("ms_rhs_fast.cu", {"MS_TMA_KEEP": 2}),
    "keep4": ("ms_rhs_fast.cu", {"MS_TMA_KEEP": 4}),
    "keep6": ("ms_rhs_fast.cu", {"MS_TMA_KEEP": 6}),
    "tcs_old": ("ms_batch.cu", {"MS_T2_SREC": 0, "MS_T2_END_RELAXED": 0, "MS_TC_PACKED": 2}),
    "tcs_noepi": ("ms_batch.cu", {"MS_T2_NOEPI": 1, "MS_T2_SREC": 0}),
    "tcs_p3_nosrec": ("ms_batch.cu", {"MS_T2_SREC": 0}),
    "tcs_p2": ("ms_batch.cu", {"MS_TC_PACKED": 2}),
    "tcx_nostore": ("ms_batch.cu", {"MS_T2_EXP_EPI": 1}),
    "tcx_norec": ("ms_batch.cu", {"MS_T2_EXP_EPI": 2}),
    "tcx_notmem": ("ms_batch.cu", {"MS_T2_EXP_EPI": 3}),
    "pf_t384": ("ms_rhs_fast.cu", {"MS_PK_PREFETCH": 1, "MS_FAST_THREADS": 384}),
    "pf_t256": ("ms_rhs_fast.cu", {"MS_PK_PREFETCH": 1, "MS_FAST_THREADS": 256}),
    "pf_r4": ("ms_rhs_fast.cu", {"MS_PK_PREFETCH": 1, "MS_FAST_R": 4}),
    "pf_r6_t384": ("ms_rhs_fast.cu", {"MS_PK_PREFETCH": 1, "MS_FAST_R": 6, "MS_FAST_THREADS": 384}),
    "t384": ("ms_rhs_fast.cu", {"MS_FAST_THREADS": 384}),
    "r12_t384": ("ms_rhs_fast.cu", {"MS_FAST_R": 12, "MS_FAST_THREADS": 384}),
}


def main(names=None):
    B.build_library()
    out = B.PKG / "_variants"
    out.mkdir(exist_ok=True)
    nvcc = B._nvcc()

    def one(item):
        name, (tu, defs) = item
        obj = out / f"{tu}_{name}.o"
        lib = out / f"lib_{name}.so"
        dflags = [f"-D{k}={v}" for k, v in defs.items()]
        subprocess.run([nvcc, *B._host_cxx(), *B.NVCC_FLAGS, *dflags, "-I", str(ROOT / "include"), "-c",
                        str(B.CSRC / tu), "-o", str(obj)], check=True)
        others = [str(B.BUILD / (src + ".o")) for src in B.SOURCES if src != tu]
        subprocess.run([nvcc, *B._host_cxx(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(lib),
                        *others, str(obj), "-lcudadevrt"], check=True)
        return name

    items = [(k, v) for k, v in VARIANTS.items() if not names or k in names]
    with ThreadPoolExecutor(8) as ex:
        for n in ex.map(one, items):
            print("built", n)


if __name__ == "__main__":
    main(sys.argv[1:])
