"""GPU command line with the reference's contract (cli.py): the same
subcommand names, options, output files (.mosst payloads, JSON sidecars and
``<out>.manifest.json``), echo lines and exit codes, with the quantizer and
the GEMM running on the B200 kernels.

    python -m paper_2511_05811_b200.cli quantize --scheme mx2 --in x.mosst --out q.mosst --meta q.json
    python -m paper_2511_05811_b200.cli gemm --m 256 --n 512 --k 1024 --scheme mx2 --verify --out r.json
    python -m paper_2511_05811_b200.cli codec-table --format e4m3

Covered: ``quantize`` (schemes ``tensor``, ``mx2`` and — through the COAT
comparator — ``group`` with group size 128; E4M3, CEIL_POW2, k2=32:
cli.py:93-133), ``gemm`` (schemes ``mx2`` and ``pergroup``, counters or
``--verify`` against the float64 dequantize-then-multiply oracle:
cli.py:221-275), ``codec-table`` (cli.py:71-90).  E5M2, NEAREST_LOG2, other
group sizes and the SNR / bound / autoscale / train simulations are not on the
MOSS hot path and exit with the reference's error convention.  Errors print a JSON line
``{"error": <class>, "message": ...}`` and exit 1 (cli.py:313-315).
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

import click
import numpy as np

from . import __version__
from .errors import MossqError
from .fp8 import E4M3, decode_table
from .tensor import DType, tensor_randn, tensor_read, tensor_write

E8M0_INVALID_CODE = 255


def _manifest(out_path, subcommand: str, config: dict, outputs: list) -> None:
    doc = {"subcommand": subcommand, "config": config, "seed": config.get("seed"), "version": __version__,
           "outputs": [str(o) for o in outputs], "device": "cuda (sm_100a kernels)"}
    Path(str(out_path) + ".manifest.json").write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def _cell(c) -> str:
    return repr(c) if isinstance(c, float) else str(c)


def _unsupported(what: str):
    raise click.ClickException(f"{what} is not on the MOSS FP8 hot path (use the reference mossq CLI)")


@click.group()
@click.version_option(__version__)
def cli():
    """B200 MOSS FP8 toolkit (reference-compatible subset)."""


@cli.command("codec-table")
@click.option("--format", "fmt_name", type=click.Choice(["e4m3", "e5m2", "e8m0"]), required=True)
@click.option("--out", type=click.Path(), default=None, help="CSV path (default stdout)")
def codec_table(fmt_name, out):
    """All code/value pairs of one format (cli.py:71-90)."""
    if fmt_name == "e8m0":
        rows = [(c, float(np.ldexp(1.0, c - 127))) for c in range(256) if c != E8M0_INVALID_CODE]
        rows.append((E8M0_INVALID_CODE, "reserved"))
    elif fmt_name == "e4m3":
        tab = decode_table(E4M3, device="cpu").numpy()
        rows = [(c, float(tab[c])) for c in range(256)]
    else:
        _unsupported("E5M2")
    lines = ["code,value"] + [",".join(_cell(v) for v in r) for r in rows]
    if out:
        Path(out).write_text("\n".join(lines) + "\n")
        _manifest(out, "codec-table", {"format": fmt_name}, [out])
        click.echo(f"wrote {out}")
    else:
        for line in lines:
            click.echo(line)


@cli.command()
@click.option("--scheme", type=click.Choice(["tensor", "group", "mx2"]), required=True)
@click.option("--format", "fmt_name", type=click.Choice(["e4m3", "e5m2"]), default="e4m3")
@click.option("--in", "in_path", type=click.Path(exists=True), required=True)
@click.option("--out", type=click.Path(), required=True, help="code payload (.mosst)")
@click.option("--meta", type=click.Path(), required=True, help="sidecar JSON")
@click.option("--group-size", type=int, default=128)
@click.option("--k2", type=int, default=32)
@click.option("--rounding", type=click.Choice(["ceil", "nearest"]), default="ceil")
def quantize(scheme, fmt_name, in_path, out, meta, group_size, k2, rounding):
    """Quantize a .mosst f32 tensor on the GPU and write codes + metadata (cli.py:93-133)."""
    from .quantize import quant_per_group, quant_per_tensor, quant_two_level
    if scheme == "group" and group_size != 128:
        _unsupported("per-group sizes other than 128")
    if fmt_name != "e4m3":
        _unsupported("E5M2")
    if rounding != "ceil" or k2 != 32:
        _unsupported("NEAREST_LOG2 / k2 != 32")
    x, tag = tensor_read(in_path)
    if tag != DType.F32:
        raise click.ClickException("input must be an f32 tensor")
    doc = {"scheme": scheme, "format": fmt_name, "shape": list(x.shape)}
    outputs = [out, meta]
    if scheme == "tensor":
        q = quant_per_tensor(x, E4M3)
        doc["scale"] = float(q.scale)
    elif scheme == "group":
        q = quant_per_group(x, E4M3, group_size=group_size)
        doc["group_size"] = group_size
        doc["scales"] = [float(v) for v in q.scales.cpu().numpy().ravel()]
        doc["scales_shape"] = list(q.scales.shape)
    else:
        q = quant_two_level(x, E4M3)
        micro_path = str(out) + ".micro.mosst"
        tensor_write(q.micro_codes, micro_path, DType.E8M0)
        doc.update({"k2": k2, "rounding": rounding, "global_scale": float(q.global_scale),
                    "micro_scales_path": micro_path})
        outputs.append(micro_path)
    tensor_write(q.codes, out, DType.FP8_E4M3)
    Path(meta).write_text(json.dumps(doc, indent=2) + "\n")
    cfg = {"scheme": scheme, "format": fmt_name, "in": str(in_path), "group_size": group_size, "k2": k2,
           "rounding": rounding}
    _manifest(out, "quantize", cfg, outputs)
    click.echo(f"wrote {out} ({scheme}, {fmt_name})")


@cli.command()
@click.option("--m", type=int, required=True)
@click.option("--n", type=int, required=True)
@click.option("--k", type=int, required=True)
@click.option("--scheme", type=click.Choice(["mx2", "pergroup"]), required=True)
@click.option("--verify", is_flag=True, help="compare against the dequantize-then-multiply oracle")
@click.option("--counters", "show_counters", is_flag=True)
@click.option("--seed", type=int, default=0, show_default=True)
@click.option("--out", type=click.Path(), required=True)
def gemm(m, n, k, scheme, verify, show_counters, seed, out):
    """One MXFP8 GEMM on tcgen05 with a JSON report (cli.py:221-275).

    W [m, k] = tensor_randn(seed) per-tensor E4M3, X [n, k] =
    tensor_randn(seed + 1) two-level MX; C = W X^T.  --verify compares with
    the float64 product of the exactly dequantized operands (gemm.py:160-209).
    """
    import torch

    from .fp8 import fp8_decode
    from .gemm import (gemm_mx_epilogue, gemm_pergroup_mainloop, mx_epilogue_counters, pergroup_mainloop_counters,
                       quantize_gemm_operands)
    from .quantize import quant_per_group
    if scheme == "mx2" and k % 32 != 0:
        raise click.ClickException("mx2 requires K divisible by 32")
    if scheme == "pergroup" and k % 128 != 0:
        raise click.ClickException("pergroup requires K divisible by 128")
    report = {"m": m, "n": n, "k": k, "scheme": scheme, "seed": seed}
    ctr = mx_epilogue_counters(m, n, k) if scheme == "mx2" else pergroup_mainloop_counters(m, n, k)
    if verify and scheme == "pergroup":
        # the COAT-style comparator (csrc/pergroup.cu); checker: float64 product of the dequantized groups
        qa = quant_per_group(tensor_randn([m, k], seed=seed))
        qb = quant_per_group(tensor_randn([n, k], seed=seed + 1))
        outm, ctr = gemm_pergroup_mainloop(qa, qb)
        deq = lambda q, r: (fp8_decode(q.codes).double().view(r, k // 128, 128)
                            * q.scales.double()[..., None]).view(r, k)
        oracle = deq(qa, m) @ deq(qb, n).t()
        diff = outm.double() - oracle
        denom = float(torch.linalg.norm(oracle))
        report["max_rel_error"] = float((diff.abs() / oracle.abs().clamp_min(1e-30)).max())
        report["frobenius_rel_error"] = float(torch.linalg.norm(diff)) / denom if denom else 0.0
    elif verify:
        w = tensor_randn([m, k], seed=seed)
        x = tensor_randn([n, k], seed=seed + 1)
        ops = quantize_gemm_operands(w, x)
        outm, ctr = gemm_mx_epilogue(ops)
        # checker: float64 product of the exactly dequantized codes (gemm.py:178-209; not the product path)
        wd = fp8_decode(ops.qw.codes).double() * float(ops.qw.scale)
        qx = ops.qx
        eff = float(qx.global_scale) * torch.ldexp(torch.ones_like(qx.micro_codes, dtype=torch.float64),
                                                   qx.micro_codes.to(torch.int64) - 127)
        xd = (fp8_decode(qx.codes).double().view(n, k // 32, 32) * eff[..., None]).view(n, k)
        oracle = wd @ xd.t()
        diff = outm.double() - oracle
        denom = float(torch.linalg.norm(oracle))
        report["max_rel_error"] = float((diff.abs() / oracle.abs().clamp_min(1e-30)).max())
        report["frobenius_rel_error"] = float(torch.linalg.norm(diff)) / denom if denom else 0.0
    report["counters"] = dataclasses.asdict(ctr)
    Path(out).write_text(json.dumps(report, indent=2) + "\n")
    _manifest(out, "gemm", {"m": m, "n": n, "k": k, "scheme": scheme, "verify": verify,
                            "counters": show_counters, "seed": seed}, [out])
    msg = f"{scheme} {m}x{n}x{k}"
    if verify:
        msg += f" frobenius_rel_error={report['frobenius_rel_error']:.3e}"
    if show_counters:
        msg += f" counters={report['counters']}"
    click.echo(msg)


def main() -> None:
    """Entry point with the reference's error convention (cli.py:307-319): one
    JSON line {"error", "message"} on stderr and a non-zero exit."""
    try:
        cli(standalone_mode=False)
    except click.exceptions.Exit as exc:
        sys.exit(exc.exit_code)
    except click.ClickException as exc:
        click.echo(json.dumps({"error": type(exc).__name__, "message": exc.format_message()}), err=True)
        sys.exit(exc.exit_code or 1)
    except click.exceptions.Abort:
        sys.exit(130)
    except MossqError as exc:
        click.echo(json.dumps({"error": type(exc).__name__, "message": str(exc)}), err=True)
        sys.exit(1)


if __name__ == "__main__":
    main()
