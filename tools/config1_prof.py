"""cProfile of the config-1 load-stepping study (host overhead per outer iteration)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import config1_time as c1  # noqa: E402

c1.run(c1.mm)
pr = cProfile.Profile()
pr.enable()
study, dt = c1.run(c1.mm)
pr.disable()
print(f"{study.state.outer_iter} outer iterations, {dt * 1e3:.1f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
