"""Critical-path trace of single-CTA rounds (INET_TRACE development build).

    make -C paper_1404_0076_b200/csrc NVFLAGS="$NVFLAGS -DINET_TRACE" OUT=tools/libinetb200_trace.so
    INET_B200_LIB=tools/libinetb200_trace.so INET_B200_CACHE=/tmp/trc INET_B200_TRACE_R0=800 \
        python tools/mtrace.py fib18

Prints, per traced round, the thread-0 view (loop top -> barrier arrive / exit)
and every working thread's split in clock cycles.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_0076_b200 import EngineConfig, evaluate  # noqa: E402
from inet.bench import program  # noqa: E402

spec = {"a38": ("ackermann", (3, 8)), "a36": ("ackermann", (3, 6)), "fib18": ("fibonacci", (18,)),
        "add": ("addition", (300, 200))}[sys.argv[1]]
p = program(spec[0])
fast = os.environ.get("FAST") == "1"  # the fast tiers (no stamps) instead of the default evaluation order
res = evaluate(p.build_input(*spec[1]), p.rules, EngineConfig(ctas_per_net=1, threads=int(os.environ.get("T", "256")),
                                                               reference_order=False if fast else None))
print("interactions", res.total_interactions, "loops", len(res.loops), flush=True)
