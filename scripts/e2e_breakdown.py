"""Where the e2e drop-in step's time goes (cfg2, S1, load steps 4..13): push, device step,
write-back (pulls + GP strain), measured with perf_counter around each part."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2209_07969_b200 import configs as C, schemes  # noqa: E402


def main():
    case = C.get_case(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
    pb = C.setup(case, C.b200_api())
    kind = schemes.SchemeKind("S1")
    for _ in range(3):
        schemes.staggered_step(pb.disc, pb.state, kind, pb.bcs, pb.params, pb.config, pb.pins)
    sess = schemes.session_for(pb.disc, pb.params, pb.config)
    t = {"push": 0.0, "step": 0.0, "write_back": 0.0, "total": 0.0}
    wb = {}
    orig = schemes._write_back
    for _ in range(10):
        t0 = time.perf_counter()
        gp = pb.state.gp
        sess.push(u=pb.state.u, d=pb.state.d, d_prev=pb.state.d_prev, psi_max=gp.psi_max)
        t1 = time.perf_counter()
        sess.step(kind, pb.bcs, pb.pins)
        t2 = time.perf_counter()
        orig(sess, pb.state)
        t3 = time.perf_counter()
        t["push"] += t1 - t0
        t["step"] += t2 - t1
        t["write_back"] += t3 - t2
        t["total"] += t3 - t0
    print({k: round(v * 100, 3) for k, v in t.items()}, "ms per step")
    # write-back parts
    nn, ne = sess.n_nodes, sess.n_elems
    for name, fn in [
        ("pull u,d,psi_max in place", lambda: sess.pull_into(u=pb.state.u, d=pb.state.d,
                                                            psi_max=pb.state.gp.psi_max)),
        ("pull d_prev+3 GP pinned", lambda: sess.pull_into(
            d_prev=schemes.N.PINNED.empty((nn,)), tr_eps_plus=schemes.N.PINNED.empty((ne, 4)),
            dev_dot_dev=schemes.N.PINNED.empty((ne, 4)), psi_plus=schemes.N.PINNED.empty((ne, 4)))),
        ("gp_strain pinned", lambda: sess.gp_strain(pinned=True)),
        ("push u,d,d_prev,psi_max", lambda: sess.push(u=pb.state.u, d=pb.state.d,
                                                      d_prev=pb.state.d_prev,
                                                      psi_max=pb.state.gp.psi_max)),
        ("push pinned copies", None),
    ]:
        if fn is None:
            pu = schemes.N.PINNED.empty(pb.state.u.shape); pu[...] = pb.state.u
            pdd = schemes.N.PINNED.empty(pb.state.d.shape); pdd[...] = pb.state.d
            pm = schemes.N.PINNED.empty(pb.state.gp.psi_max.shape); pm[...] = pb.state.gp.psi_max
            fn = lambda: sess.push(u=pu, d=pdd, d_prev=pb.state.d_prev, psi_max=pm)  # noqa: E731
        fn()
        t0 = time.perf_counter()
        for _ in range(10):
            fn()
        print(f"{name:32s} {(time.perf_counter() - t0) * 100:.3f} ms")


if __name__ == "__main__":
    main()
