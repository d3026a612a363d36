"""Run `steps` ETD2RK-DS steps of a BASELINE config (optionally at reduced n) — a
small, deterministic command for ncu captures: python tools/one_step.py CFG [N] [STEPS] [--thomas]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06849_b200 import configs  # noqa: E402

kw = {}
if "--thomas" in sys.argv:
    sys.argv.remove("--thomas")
    from paper_2601_06849_b200 import etd

    kw["backend"] = etd.BackendKind.Thomas
cfg = configs.CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
plan = configs.make_plan(cfg, n, **kw)
for s, a in enumerate(configs.initial_state(cfg, n)):
    plan.upload(s, a)
plan.step(steps)
u, nn, t = plan.download(0)
print(f"cfg{cfg.id} n={n} steps={nn} t={t:.4f} u[0]={u[0]:.6e}")
