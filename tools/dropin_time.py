"""Host-side cost of the drop-in entry point (graph -> SolveReport) per phase, first and cached calls.

python tools/dropin_time.py [cfg ...]
"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_2512_02293_b200 import solver as S  # noqa: E402
from paper_2512_02293_b200.device import DeviceProblem, HostLayout  # noqa: E402
from paper_2512_02293_b200.problem import options_dict, write_back  # noqa: E402
from paper_2512_02293_b200.types import SolveOptions  # noqa: E402
from paper_2512_02293_b200.workloads import CONFIGS, make_workload  # noqa: E402


def main(cfgs):
    for cfg in cfgs:
        g = make_workload(cfg)
        opts = SolveOptions(max_iterations=CONFIGS[cfg].iterations)
        o = options_dict(opts)
        for rep in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            H = HostLayout.from_graph(g, o)
            t1 = time.perf_counter()
            if rep == 0:
                dp = DeviceProblem(None, o, layout=H)
            else:
                dp.rebind(H)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            r = dp.solve()
            t3 = time.perf_counter()
            s = dp.download()
            g2 = g  # write back into the same graph objects (timing only)
            write_back(g2, s["q"], s["p"], s["v"], s["bg"], s["ba"], s["disp"], s["grav_q"], opts)
            t4 = time.perf_counter()
            print(f"cfg{cfg} call {rep}: layout {1e3 * (t1 - t0):.1f} ms, "
                  f"{'create' if rep == 0 else 'rebind'}+upload {1e3 * (t2 - t1):.1f} ms, solve {1e3 * (t3 - t2):.1f} ms, "
                  f"download+write-back {1e3 * (t4 - t3):.1f} ms; host overhead {1e3 * ((t4 - t0) - (t3 - t2)):.1f} ms "
                  f"({r['iterations']} it)", flush=True)
            g = make_workload(cfg)
        dp.close()
        # the public call end to end (cache warm after the first)
        for rep in range(3):
            g = make_workload(cfg)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            S.solve_vi_ba(g, opts)
            t1 = time.perf_counter()
            print(f"cfg{cfg} solve_vi_ba call {rep}: {1e3 * (t1 - t0):.1f} ms", flush=True)
        S.clear_cache()


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 4])
