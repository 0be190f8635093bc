import sys, collections
sys.path.insert(0, "/root/repo")
from paper_2605_23727_b200 import harness as H
from paper_2605_23727_b200 import solver as S
cases = []
tid = 3000
for n in (50, 100):
    for tol in (1e-3, 1e-4, 1e-5, 1e-6):
        for kc in (0.001, 0.1, 1.0):
            for i0 in (0.228249, 1.5):
                cases.append(H.TestCase(test_id=tid, benchmark="cc", agents=n, rel_tol=tol, abs_tol=1e-2*tol, t_final=48.0, coupling_k=kc, stimulus_i0=i0)); tid += 1
rows = H.run_cases(cases, opt=H.RunOptions(time_limits=False))
cnt = collections.Counter((r.variant, r.rel_tol, S.SolveStatus(r.status).name) for r in rows if r.status != 0)
for k, v in sorted(cnt.items()): print(k, v)
