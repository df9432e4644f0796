"""In-process A/B of libkmb200.so builds (same ABI, different compile-time options).

    python tools/ab_probe.py paper_2103_01691_b200/libkmb200.so build/ab1/libkmb200.so ...

Every library is loaded side by side (ctypes), gets its own stream-K workspace on the
current stream, and runs the same km_mumode launches on the same device buffers; the
rounds alternate between the libraries so box-to-box and clock drift cancel.  Prints
the median µs per launch per case and library, and whether the outputs are bitwise equal
to the first library's.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2103_01691_b200 import _native  # noqa: E402

DEV = torch.device("cuda", 0)
F64, C128 = _native.KM_F64, _native.KM_C128


def load(path):
    h = ctypes.CDLL(os.path.abspath(path))
    _native._declare(h)
    nb = ctypes.c_size_t(0)
    _native.check(h.km_stream_workspace_bytes(ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=DEV)
    raw = torch.cuda.current_stream().cuda_stream
    assert h.km_set_stream_workspace(ctypes.c_void_p(raw), ctypes.c_void_p(ws.data_ptr()), nb.value) == 0
    return h, ws


def case(name, u_dt, l_dt, m, nl, nmu, nr):
    g = torch.Generator(device=DEV).manual_seed(0)
    tdt = torch.complex128 if u_dt == C128 else torch.float64
    ldt = torch.complex128 if l_dt == C128 else torch.float64
    odt = torch.complex128 if C128 in (u_dt, l_dt) else torch.float64
    u = torch.randn(nl * nmu * nr, dtype=tdt, device=DEV, generator=g)
    L = torch.randn(m * nmu, dtype=ldt, device=DEV, generator=g) / nmu ** 0.5
    flop = (2 if odt == torch.float64 else (8 if (u_dt == C128 and l_dt == C128) else 4)) * m * nl * nmu * nr
    return dict(name=name, u=u, ud=u_dt, L=L, ld=l_dt, m=m, nl=nl, nmu=nmu, nr=nr, odt=odt, flop=flop)


CASES = [
    case("pipe f64 dir1 1024^2", F64, F64, 1024, 1, 1024, 1024),
    case("pipe f64 dir2 1024^2", F64, F64, 1024, 1024, 1024, 1),
    case("c128 x f64 dir2 1024^2", C128, F64, 1024, 1024, 1024, 1),
    case("c128 x f64 dir2 256^3", C128, F64, 256, 256, 256, 256),
    case("c128 dir1 256^3", C128, C128, 256, 1, 256, 65536),
    case("c128 dir3 256^3", C128, C128, 256, 65536, 256, 1),
    case("f64 dir2 512^3", F64, F64, 512, 512, 512, 512),
]


def run(h, c, out, reps):
    args = (ctypes.c_void_p(c["u"].data_ptr()), c["ud"], ctypes.c_void_p(c["L"].data_ptr()), c["ld"],
            ctypes.c_void_p(out.data_ptr()), c["m"], c["nl"], c["nmu"], c["nr"], None,
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        rc = h.km_mumode(*args)
    e1.record()
    e1.synchronize()
    assert rc == 0, (h.km_last_error() or b"").decode()
    return e0.elapsed_time(e1) / reps * 1e3


def main(paths, rounds=5, reps=20):
    libs = [load(p) for p in paths]
    print("libs:", paths)
    for c in CASES:
        outs = [torch.empty(c["m"] * c["nl"] * c["nr"], dtype=c["odt"], device=DEV) for _ in libs]
        for (h, _), o in zip(libs, outs):
            run(h, c, o, 3)
        times = [[] for _ in libs]
        for _ in range(rounds):
            for i, (h, _) in enumerate(libs):
                times[i].append(run(h, c, outs[i], reps))
        same = [bool(torch.equal(outs[0], o)) for o in outs]
        if os.environ.get("AB_CHECK") == "1":  # relative error against a torch float64/complex128 product
            L = c["L"].view(c["m"], c["nmu"])
            ref = torch.einsum("ik,rkl->ril", L.to(c["odt"]), c["u"].view(c["nr"], c["nmu"], c["nl"]).to(c["odt"]))
            errs = [float((o.view_as(ref) - ref).abs().max() / ref.abs().max()) for o in outs]
            print("   max rel err", ["%.1e" % e for e in errs])
        med = [sorted(t)[len(t) // 2] for t in times]
        print(f"{c['name']:26s} " + "  ".join(f"{m:8.1f} us ({c['flop'] / m / 1e6:5.1f} TF)" for m in med)
              + f"  bitwise-equal {same}", flush=True)


if __name__ == "__main__":
    # AB_ONCE=1: one launch per case and library (for ncu captures); AB_CASES=substring filter
    once = os.environ.get("AB_ONCE") == "1"
    if os.environ.get("AB_CASES"):
        CASES[:] = [c for c in CASES if any(k in c["name"] for k in os.environ["AB_CASES"].split(","))]
    main(sys.argv[1:] or [os.path.join("paper_2103_01691_b200", "libkmb200.so")],
         rounds=1 if once else 5, reps=1 if once else 20)
