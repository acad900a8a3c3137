"""``fit`` command of the reference CLI (cpfast/cli.py:95-134) on the B200 engine.

    python -m paper_1205_2584_b200.cli fit TENSOR.cptn --rank R [--algo auto|flm-a|flm-b]
        [--tau T] [--tol T] [--max-iters K] [--seed S] [--init svd|random] [--truth META] [--out P]

    python -m paper_1205_2584_b200.cli bench --dims 20,20,20 --rank 3 --nu 0.1,0.9 --snr inf --algos auto
        --seeds 10 [--complex] [--tol T] [--max-iters K] [--out bench.csv]

Same options, defaults, output lines, factor files (``P_factor<n>.cptn``) and CSV records as the
reference's ``fit`` (cli.py:95-134) and ``bench`` (cli.py:137-175).  The tensor file is streamed
straight into device memory (``fit_file``); variants other than the fast damped Gauss-Newton ones
exit with an error (``fit``) or become 'error' records (``bench``): the B200 backend has no CPU
fallback.  The reference's ``gen`` / ``spectrum`` / ``verify`` commands are test scaffolding
outside the hot path and are not provided.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import click

from . import cptn
from .records import record_from_result, write_csv
from .solver import VARIANTS, FitConfig, fit_file
from .tensor import KruskalModel


def _load_truth(meta_path) -> KruskalModel:
    meta = cptn.read_metadata(meta_path)
    return KruskalModel([cptn.read_matrix(p) for p in meta["factors"].split(";")])


@click.group()
def main():
    """CP decomposition on the B200 engine."""


@main.command("fit")
@click.argument("tensor_file", type=click.Path(exists=True))
@click.option("--algo", type=click.Choice(VARIANTS), default="auto", show_default=True)
@click.option("--rank", "-r", type=int, required=True)
@click.option("--tau", type=float, default=1e-3, show_default=True)
@click.option("--tol", type=float, default=1e-8, show_default=True)
@click.option("--max-iters", type=int, default=1000, show_default=True)
@click.option("--seed", type=int, default=0, show_default=True)
@click.option("--init", type=click.Choice(["svd", "random"]), default="svd")
@click.option("--truth", default=None, type=click.Path(exists=True),
              help="Metadata sidecar of the generating run, for MedSAE scoring.")
@click.option("--out", default=None, help="Prefix for fitted factors + CSV record.")
@click.option("--device", type=int, default=0, show_default=True, help="CUDA device.")
def cmd_fit(tensor_file, algo, rank, tau, tol, max_iters, seed, init, truth, out, device):
    """Decompose a tensor file with the selected algorithm."""
    config = FitConfig(rank=rank, variant=algo, tau=tau, tol=tol, max_iters=max_iters, seed=seed, init=init)
    try:
        result = fit_file(tensor_file, config, device=device)
    except ValueError as exc:  # unsupported variant / malformed file: reported, exit status 1
        click.echo(str(exc), err=True)
        sys.exit(1)
    truth_model = _load_truth(truth) if truth else None
    record = record_from_result(result, truth_model, seed, float("nan"), rank, None, algo)
    click.echo(f"algo={algo} iters={record.iters} accepted={record.accepted_iters} "
               f"relerr={record.final_relerr:.3e} stop={record.stop_reason} time_ms={record.time_ms:.1f}")
    if out:
        for n, factor in enumerate(result.model.factors, start=1):
            cptn.write_matrix(f"{out}_factor{n}.cptn", factor)
        write_csv(f"{out}.csv", [record])
        click.echo(f"wrote {out}.csv")
    if record.stop_reason == "error":
        sys.exit(1)


def _ints(text: str) -> tuple:
    return tuple(int(p) for p in text.split(",") if p.strip())


def _floats(text: str) -> tuple:
    return tuple(float("inf") if p.strip().lower() in ("inf", "none") else float(p)
                 for p in text.split(",") if p.strip())


@main.command("bench")
@click.option("--dims", default="20,20,20", show_default=True)
@click.option("--rank", default="3", show_default=True, help="Comma-separated ranks.")
@click.option("--nu", default="0.1,0.9", show_default=True)
@click.option("--snr", default="inf", show_default=True)
@click.option("--algos", default="als-ls,auto", show_default=True)
@click.option("--seeds", type=int, default=10, show_default=True)
@click.option("--complex", "use_complex", is_flag=True)
@click.option("--tol", type=float, default=1e-8, show_default=True)
@click.option("--max-iters", type=int, default=1000, show_default=True)
@click.option("--out", default="bench.csv", show_default=True)
def cmd_bench(dims, rank, nu, snr, algos, seeds, use_complex, tol, max_iters, out):
    """Monte-Carlo sweep over (nu, R, SNR) x seeds x algorithms."""
    from . import gridbench
    from .tensor import COMPLEX, REAL

    algo_list = tuple(a.strip() for a in algos.split(",") if a.strip())
    snr_list = tuple(None if math.isinf(v) else v for v in _floats(snr))
    records = gridbench.run_grid(_ints(dims), _ints(rank), _floats(nu), snr_list, algo_list, seeds,
                                 COMPLEX if use_complex else REAL, tol=tol, max_iters=max_iters)
    write_csv(out, records)
    summary = gridbench.summarize(records)
    summary_path = str(Path(out).with_name(Path(out).stem + "_summary.csv"))
    gridbench.write_summary_csv(summary_path, summary)
    click.echo(f"wrote {len(records)} rows to {out}; summary in {summary_path}")
    for row in summary:
        click.echo(f"nu={row['nu']} R={row['R']} snr={row['snr_db']} algo={row['algo']}: "
                   f"median_iters={row['median_iters']} median_relerr={row['median_relerr']}")


if __name__ == "__main__":
    main()
