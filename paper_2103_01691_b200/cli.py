"""Command line over the device drivers, with the reference's report schema.

Same subcommands, flags, defaults, exit codes (0 ok, 1 numerical / I/O
failure, 2 usage) and CSV / JSON / table output as the reference's
``kronmode.cli`` (cli.py:29-32 columns, 114-176 parser, 268-331 rendering),
so its CLI tests and any script that parses its reports keep working; the
runs themselves go through :mod:`drivers`, i.e. the GPU hot path.  One flag
is added: ``--device cuda:N`` selects the GPU.

``selftest`` runs the reference's five built-in equivalence checks against
the device implementation.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
from dataclasses import dataclass, field, fields

import numpy as np

from . import drivers
from .errors import KronmodeError

__all__ = ["CSV_COLUMNS", "CliConfig", "build_parser", "main", "parse_args", "run"]

CSV_COLUMNS = ("problem", "n", "k", "p", "steps", "tau", "precision", "norm",
               "rel_error", "time_exp_s", "time_mumode_s", "time_other_s", "total_s")

_GRID = ("heat", "pipeflow", "gpe")
_HERMITE = ("schrodinger-ti", "schrodinger-td")


@dataclass
class CliConfig:
    command: str
    n: int | None = None
    n_list: list = field(default_factory=list)
    k: int | None = None
    k_list: list = field(default_factory=list)
    p: float | None = None
    T: float | None = None
    steps: int | None = None
    tau: float | None = None
    k_ref: int | None = None
    ref_steps: int | None = None
    problem: str | None = None
    precision: str = "double"
    norm: str = "max"
    output: str = "table"
    out_path: str | None = None
    seed: int = 1234
    threads: int | None = None
    device: str | None = None


# ---------------------------------------------------------------------------
# argument types (cli.py:59-93)


def _type(fn):
    def parse(text):
        try:
            return fn(text)
        except (ValueError, TypeError) as exc:
            raise argparse.ArgumentTypeError(str(exc) or f"bad value {text!r}") from None
    return parse


def _pos_int_raw(text):
    try:
        v = int(text)
    except ValueError:
        raise ValueError(f"expected an integer, got {text!r}") from None
    if v <= 0:
        raise ValueError(f"expected a positive integer, got {text!r}")
    return v


def _pos_float_raw(text):
    try:
        v = float(text)
    except ValueError:
        raise ValueError(f"expected a number, got {text!r}") from None
    if not (v > 0 and math.isfinite(v)):
        raise ValueError(f"expected a positive number, got {text!r}")
    return v


def _order_raw(text):
    if text.strip().lower() in ("inf", "spectral"):
        return math.inf
    v = _pos_int_raw(text)
    if v % 2:
        raise ValueError(f"expected an even order or 'inf', got {text!r}")
    return v


def _list_raw(text):
    try:
        vals = [int(t) for t in text.split(",") if t.strip()]
    except ValueError:
        raise ValueError(f"expected comma-separated integers, got {text!r}") from None
    if not vals or min(vals) <= 0:
        raise ValueError(f"expected positive integers, got {text!r}")
    return vals


POS_INT, POS_FLOAT, ORDER, INT_LIST = map(_type, (_pos_int_raw, _pos_float_raw, _order_raw, _list_raw))

# (flag, dest, type, default, help) per subcommand; defaults as cli.py:114-169
_SPECS = {
    "heat": ("periodic 3D heat equation with analytic reference", [
        ("--n", "n", POS_INT, 40, "grid points per direction"),
        ("--p", "p", ORDER, 2, "even finite-difference order, or 'inf' for spectral"),
        ("--T", "T", POS_FLOAT, 1.0, "final time"),
        ("--steps", "steps", POS_INT, 1, "number of time steps")]),
    "pipeflow": ("2D pipe diffusion-advection vs Arnoldi baseline", [
        ("--n", "n", POS_INT, 32, "grid points per direction"),
        ("--T", "T", POS_FLOAT, 4.0, "final time"),
        ("--steps", "steps", POS_INT, 1, "number of time steps")]),
    "schrodinger-ti": ("Schrodinger equation, time-independent potential, Hermite basis", [
        ("--k", "k", POS_INT, 40, "basis functions per direction"),
        ("--T", "T", POS_FLOAT, 1.0, "final time"),
        ("--k-ref", "k_ref", POS_INT, 120, "reference resolution for the error (0 disables)")]),
    "schrodinger-td": ("Schrodinger equation, driven potential, midpoint Magnus stepping", [
        ("--k", "k", POS_INT, 20, "basis functions per direction"),
        ("--T", "T", POS_FLOAT, 1.0, "final time"),
        ("--steps", "steps", POS_INT, 32, "number of time steps"),
        ("--ref-steps", "ref_steps", POS_INT, 2048, "reference step count for the error (0 disables)")]),
    "gpe": ("Gross-Pitaevskii vortex pair with Strang splitting", [
        ("--n", "n", POS_INT, 32, "grid points per direction"),
        ("--T", "T", POS_FLOAT, 2.5, "final time"),
        ("--tau", "tau", POS_FLOAT, 0.1, "time step size")]),
    "sweep": ("run one problem over a list of resolutions", [
        ("--n", "n_list", INT_LIST, [], "comma-separated grid sizes (grid-based problems)"),
        ("--k", "k_list", INT_LIST, [], "comma-separated basis sizes (Hermite problems)"),
        ("--p", "p", ORDER, 2, "finite-difference order (heat)"),
        ("--T", "T", POS_FLOAT, None, "final time (problem default if omitted)"),
        ("--steps", "steps", POS_INT, None, "number of time steps"),
        ("--tau", "tau", POS_FLOAT, None, "time step size (gpe)"),
        ("--k-ref", "k_ref", POS_INT, 120, "reference resolution (schrodinger-ti)"),
        ("--ref-steps", "ref_steps", POS_INT, 2048, "reference step count (schrodinger-td)")]),
    "selftest": ("run the built-in equivalence checks on the device", []),
}


def _common(sp):
    sp.add_argument("--precision", choices=("single", "double"), default="double",
                    help="scalar precision of the run (default: double)")
    sp.add_argument("--norm", choices=("max", "two"), default="max",
                    help="norm of the reported relative error (default: max)")
    sp.add_argument("--output", choices=("csv", "json", "table"), default="table",
                    help="report format (default: table)")
    sp.add_argument("--out", dest="out_path", default=None, metavar="PATH",
                    help="write the report to PATH instead of stdout")
    sp.add_argument("--seed", type=int, default=1234, help="seed of the randomized self-checks")
    sp.add_argument("--threads", type=POS_INT, default=None,
                    help="host BLAS worker hint for the host-side setup (default: KRONMODE_THREADS)")
    sp.add_argument("--device", default=None, metavar="cuda[:N]",
                    help="CUDA device of the run (default: the current device)")


def build_parser():
    parser = argparse.ArgumentParser(
        prog="kronmode-b200",
        description="Benchmarks of the mode-wise exponential integrator, run on the B200 hot path.")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (help_text, options) in _SPECS.items():
        sp = sub.add_parser(name, help=help_text)
        if name == "sweep":
            sp.add_argument("--problem", choices=_GRID[:2] + _HERMITE + _GRID[2:], required=True)
        for flag, dest, typ, default, h in options:
            sp.add_argument(flag, dest=dest, type=typ, default=default, help=h)
        _common(sp)
    return parser


def parse_args(argv):
    """Parse and validate (cli.py:172-195); usage errors exit with code 2."""
    parser = build_parser()
    ns = parser.parse_args(argv)
    names = {f.name for f in fields(CliConfig)}
    cfg = CliConfig(**{k: v for k, v in vars(ns).items() if k in names})
    if cfg.threads is None and "KRONMODE_THREADS" in os.environ:
        env = os.environ["KRONMODE_THREADS"]
        try:
            cfg.threads = _pos_int_raw(env)
        except ValueError:
            parser.error(f"KRONMODE_THREADS must be a positive integer, got {env!r}")
    if cfg.command == "sweep":
        grid = cfg.problem in _GRID
        if not (cfg.n_list if grid else cfg.k_list):
            parser.error(f"sweep over {cfg.problem} needs {'--n' if grid else '--k'} with at least one value")
    return cfg


# ---------------------------------------------------------------------------
# execution


_threads_ctl = None


def _setup(cfg):
    global _threads_ctl
    if cfg.threads is not None:
        try:
            from threadpoolctl import threadpool_limits
        except ImportError:  # a hint only
            pass
        else:
            _threads_ctl = threadpool_limits(limits=cfg.threads)
    if cfg.device is not None:
        from . import _device as dv

        dev = dv.torch.device(cfg.device)
        if dev.type != "cuda":
            raise KronmodeError(f"--device must name a CUDA device, got {cfg.device!r}")
        dv.torch.cuda.set_device(dev)


def _one(cfg):
    c = cfg.command
    if c == "heat":
        return drivers.heat3d_run(cfg.n, p=cfg.p, T=cfg.T, steps=cfg.steps, norm_kind=cfg.norm,
                                  precision=cfg.precision)
    if c == "pipeflow":
        return drivers.pipeflow_run(cfg.n, T=cfg.T, steps=cfg.steps, norm_kind=cfg.norm, precision=cfg.precision)
    if c == "schrodinger-ti":
        return drivers.hkp_run(cfg.k, T=cfg.T, k_ref=cfg.k_ref or None, norm_kind=cfg.norm,
                               precision=cfg.precision)
    if c == "schrodinger-td":
        return drivers.hkmp_run(cfg.k, T=cfg.T, steps=cfg.steps, ref_steps=cfg.ref_steps or None,
                                norm_kind=cfg.norm, precision=cfg.precision)
    if c == "gpe":
        return drivers.gpe_run(cfg.n, T=cfg.T, tau=cfg.tau, precision=cfg.precision)
    raise KronmodeError(f"unhandled command {c!r}")


_PROBLEM_DEFAULTS = {  # cli.py:221-227
    "heat": {"T": 1.0, "steps": 1},
    "pipeflow": {"T": 4.0, "steps": 1},
    "schrodinger-ti": {"T": 1.0},
    "schrodinger-td": {"T": 1.0, "steps": 32},
    "gpe": {"T": 2.5, "tau": 0.1},
}


def _sweep(cfg):
    grid = cfg.problem in _GRID
    out = []
    for value in (cfg.n_list if grid else cfg.k_list):
        entry = CliConfig(command=cfg.problem, p=cfg.p, T=cfg.T, steps=cfg.steps, tau=cfg.tau, k_ref=cfg.k_ref,
                          ref_steps=cfg.ref_steps, precision=cfg.precision, norm=cfg.norm, seed=cfg.seed)
        for key, default in _PROBLEM_DEFAULTS[cfg.problem].items():
            if getattr(entry, key) is None:
                setattr(entry, key, default)
        if grid:
            entry.n = value
        else:
            entry.k = value
        out.append(_one(entry))
    return out


# ---------------------------------------------------------------------------
# rendering (cli.py:250-331)


def _row(report):
    d = report.as_dict()
    p = d["p"]
    if isinstance(p, float) and p.is_integer():
        p = int(p)
    src = {"norm": "norm_kind", "rel_error": "error"}
    return {col: (p if col == "p" else d[src.get(col, col)]) for col in CSV_COLUMNS}


def _csv_cell(v):
    if v is None:
        return ""
    if isinstance(v, float):
        return "inf" if math.isinf(v) else format(v, ".15e")
    return str(v)


def _table_cell(v):
    if v is None:
        return "-"
    if isinstance(v, float):
        return "inf" if math.isinf(v) else format(v, ".3e")
    return str(v)


def render(reports, fmt, single):
    if fmt == "json":
        data = reports[0].as_dict() if single else [r.as_dict() for r in reports]
        return json.dumps(data, indent=2) + "\n"
    rows = [_row(r) for r in reports]
    if fmt == "csv":
        return "\n".join([",".join(CSV_COLUMNS)] + [",".join(_csv_cell(r[c]) for c in CSV_COLUMNS)
                                                   for r in rows]) + "\n"
    cells = [[_table_cell(r[c]) for c in CSV_COLUMNS] for r in rows]
    widths = [max([len(h)] + [len(row[i]) for row in cells]) for i, h in enumerate(CSV_COLUMNS)]
    lines = ["  ".join(h.ljust(w) for h, w in zip(CSV_COLUMNS, widths))]
    lines += ["  ".join(v.ljust(w) for v, w in zip(row, widths)) for row in cells]
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# selftest (cli.py:356-421): the same five checks, through the device path


def _selftest(cfg):
    from . import (
        KroneckerOp,
        arnoldi_expmv,
        assemble_full,
        forward_transform,
        heat_factors,
        hermite_basis,
        inverse_transform,
        matexp,
        mu_mode_product,
        norm,
        prepare,
        step,
    )

    rng = np.random.default_rng(cfg.seed)

    def index_formula():
        u, mat = rng.standard_normal((3, 4, 2)), rng.standard_normal((5, 4))
        err = np.abs(mu_mode_product(u, mat, 2) - np.einsum("ij,ajb->aib", mat, u)).max()
        assert err < 1e-13, "mode product disagrees with the index formula"

    def dense_exponential():
        for _ in range(10):
            dims = [int(rng.integers(2, 6)) for _ in range(int(rng.integers(2, 4)))]
            op = KroneckerOp(tuple(rng.standard_normal((m, m)) for m in dims))
            u = np.asfortranarray(rng.standard_normal(dims))
            got = step(prepare(op, 0.3), u).ravel(order="F")
            want = matexp(0.3 * assemble_full(op)) @ u.ravel(order="F")
            rel = np.linalg.norm(got - want) / np.linalg.norm(want)
            assert rel < 1e-12, f"propagator vs dense exponential: {rel:.2e}"

    def orthonormality():
        b = hermite_basis(40)
        dev = np.abs((b.phi * b.mod_weights) @ b.phi.T - np.eye(40)).max()
        assert dev < 1e-12, f"discrete orthonormality deviation {dev:.2e}"

    def round_trip():
        bases = (hermite_basis(24),) * 2
        v = rng.standard_normal((24, 24)) + 1j * rng.standard_normal((24, 24))
        rel = np.abs(inverse_transform(bases, forward_transform(bases, v)) - v).max() / np.abs(v).max()
        assert rel < 1e-11, f"transform round trip error {rel:.2e}"

    def arnoldi():
        op = heat_factors(8, 2)
        u = np.asfortranarray(rng.standard_normal((8, 8, 8)))
        want = step(prepare(op, 0.1), u)
        rel = norm(arnoldi_expmv(op, u, 0.1, tol=1e-10) - want, "two") / norm(want, "two")
        assert rel < 1e-8, f"Arnoldi baseline vs propagator: {rel:.2e}"

    checks = [("mode-product index formula", index_formula), ("propagator vs dense exponential", dense_exponential),
              ("discrete orthonormality", orthonormality), ("transform round trip", round_trip),
              ("Arnoldi baseline vs propagator", arnoldi)]
    failed = 0
    for name, fn in checks:
        try:
            fn()
            print(f"PASS  {name}")
        except AssertionError as exc:
            failed += 1
            print(f"FAIL  {name} ({exc})")
    print(f"{len(checks) - failed}/{len(checks)} checks passed")
    return 1 if failed else 0


def run(cfg):
    """Execute a parsed configuration and return the exit code (cli.py:424-451)."""
    try:
        _setup(cfg)
        if cfg.command == "selftest":
            return _selftest(cfg)
        single = cfg.command != "sweep"
        reports = [_one(cfg)] if single else _sweep(cfg)
        text = render(reports, cfg.output, single)
        if cfg.out_path is None:
            sys.stdout.write(text)
        else:
            with open(cfg.out_path, "w", encoding="utf-8") as fh:
                fh.write(text)
        return 0
    except KronmodeError as exc:
        print(f"kronmode: error: {exc}", file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"kronmode: i/o error: {exc}", file=sys.stderr)
        return 1


def main(argv=None):
    return run(parse_args(sys.argv[1:] if argv is None else argv))


if __name__ == "__main__":
    sys.exit(main())
