"""Host pass (run_initialization) time with the phase matrix on the host
(SP_FRONTEND_DEV=0), on the device (=1) and in the default mode (starts
on the host, moves when row operations turn heavy), for the Fig. 3 families and the
bench configs: the data behind the device-phase-store threshold in
frontend.cpp. Usage: python tools/frontend_threshold.py [n ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_03906_b200 import circuits, sampler  # noqa: E402


def cases(ns):
    for n in ns:
        for f in ("a", "b", "c"):
            yield f"{circuits.BENCH_FAMILIES[f]}_n{n}", circuits.bench_family(f, n)
    yield "cfg3_surface_d15", circuits.surface_code(15, 15, 1e-3)
    yield "cfg4_random_clifford", circuits.random_clifford()
    yield "surface_d25", circuits.surface_code(25, 25, 1e-3)


def main():
    ns = [int(a) for a in sys.argv[1:]] or [250, 500, 1000]
    print("case,n_sym,n_meas,host_s,dev_s,auto_s")
    for name, text in cases(ns):
        row = [name]
        ts = []
        for dev in ("0", "1", None):
            if dev is None:
                os.environ.pop("SP_FRONTEND_DEV", None)
            else:
                os.environ["SP_FRONTEND_DEV"] = dev
            t0 = time.perf_counter()
            r = sampler.run_initialization(text)
            ts.append(time.perf_counter() - t0)
        row += [str(r.n_sym), str(r.n_meas)] + [f"{t:.4f}" for t in ts]
        print(",".join(row), flush=True)


if __name__ == "__main__":
    main()
