import os, sys
sys.path.insert(0, os.getcwd())
from paper_2605_03561_b200 import Q_CUBE, Q_STATS, Context, scenarios
with Context(0) as ctx:
    ctx.generate_iterative(scenarios.device_scenario(8192, 500, spread="gamess", seed=3))
    for _ in range(4):
        info = ctx.query(Q_CUBE | Q_STATS, anchor=1)
    print(info["ms_total"], info["ms_main"], info["ms_bounds"], info["host_syncs"])
