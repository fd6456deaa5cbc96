import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, evaluate, errors
from inet.bench import program
p = program("ackermann")
for g in (0, 2):
    try:
        res = evaluate(p.build_input(2, 3), p.rules, EngineConfig(ctas_per_net=g))
        print("G", g, "ints", res.total_interactions, [(s.interactions, s.communications, s.live_equations) for s in res.loops])
    except errors.InetError as e:
        print("G", g, "error", e)
