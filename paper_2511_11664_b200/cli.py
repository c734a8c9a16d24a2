"""`sczip`-compatible command line, every data path on the GPU
(reference: cli.py:1-150).

    python -m paper_2511_11664_b200 compress   IN.rtf --q Q [--n N] -o OUT.scz [--format 2 --block-syms B]
    python -m paper_2511_11664_b200 decompress IN.scz -o OUT.rtf
    python -m paper_2511_11664_b200 analyze    IN.rtf --q Q [--csv REPORT.csv]
    python -m paper_2511_11664_b200 bench      --dims 128,28,28 --q-list 2,4,8 --csv OUT.csv [...]
    python -m paper_2511_11664_b200 latency    IN.scz [--eps --bw-hz --snr-db --sigma2]

The sub-commands, flags, SCZ_* environment defaults and exit codes
(0 ok, 1 usage error, 2 data error: ValueError / SczipError / OSError) are
the reference's, so scripts written against `sczip` keep working.
`compress`/`decompress` go through container.compress/decompress (the
libsczip_b200 C ABI), `analyze` prices every reshape candidate in one device
pass (optimizer.exhaustive_search), and `bench` sweeps through
bench.run_sweep with CUDA-event timings.  `--format 2` writes the FORMAT.md
v2 container (interleaved lanes); the default is the reference's v1 bytes.
"""

from __future__ import annotations

import argparse
import os
import sys

from . import bench, channel, container, optimizer, tensor
from .errors import SczipError

EXIT_OK, EXIT_USAGE, EXIT_DATA = 0, 1, 2

# flag -> (environment override, channel default, ChannelParams.from_db keyword)
_LINK_FLAGS = {
    "--eps": ("SCZ_EPS", channel.DEFAULT_EPS, "outage_prob"),
    "--bw-hz": ("SCZ_BW_HZ", channel.DEFAULT_BANDWIDTH_HZ, "bandwidth_hz"),
    "--snr-db": ("SCZ_SNR_DB", channel.DEFAULT_SNR_DB, "snr_db"),
    "--sigma2": ("SCZ_SIGMA2", channel.DEFAULT_FADING_VAR, "fading_var"),
}


class _UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    """argparse that reports usage errors as exit code 1 (not argparse's 2)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise _UsageError(message)


def _link_args(p: argparse.ArgumentParser) -> None:
    for flag, (env, default, _) in _LINK_FLAGS.items():
        raw = os.environ.get(env)
        p.add_argument(flag, type=float, default=float(raw) if raw is not None else default)


def _link(args) -> channel.ChannelParams:
    kw = {key: getattr(args, flag[2:].replace("-", "_")) for flag, (_, _, key) in _LINK_FLAGS.items()}
    return channel.ChannelParams.from_db(**kw)


def _int_list(text: str) -> list[int]:
    return [int(v) for v in text.split(",") if v.strip()]


# ---------------------------------------------------------------- commands
def _cmd_compress(a) -> None:
    t = tensor.read_rtf(a.input)
    c = container.compress(t, a.q, a.n, format=a.format, block_syms=a.block_syms)
    container.write_container(c, a.output)
    print(f"{a.output}: {c.total_bytes} bytes (header {c.header_bytes}, payload {c.payload_bytes}), "
          f"N={c.n_rows}, K={c.n_cols}, nnz={c.nnz}")


def _cmd_decompress(a) -> None:
    t = container.decompress(container.read_container(a.input))
    tensor.write_rtf(t, a.output)
    print(f"{a.output}: dims {'x'.join(str(d) for d in t.dims)}")


def _cmd_analyze(a) -> None:
    t = tensor.read_rtf(a.input)
    best, report = optimizer.exhaustive_search(t, a.q)
    rows = [f"{'N':>10} {'K':>8} {'entropy':>10} {'t_tot':>14} chosen"]
    for cand in report.candidates:
        flag = "*" if cand.n_rows == best else ""
        rows.append(f"{cand.n_rows:>10} {cand.n_cols:>8} {cand.entropy_bits:>10.4f} {cand.t_tot:>14.1f} {flag}")
    print("\n".join(rows))
    if a.csv:
        optimizer.write_report_csv(report, a.csv)


def _cmd_bench(a) -> None:
    t = bench.gen_synthetic(a.kind, _int_list(a.dims), a.sparsity, a.seed)
    recs = bench.run_sweep(t, _int_list(a.q_list), tensor_id=f"{a.kind}-{a.seed}", repetitions=a.repetitions,
                           csv_path=a.csv, link=_link(a))
    print(f"{a.csv}: {len(recs)} rows")


def _cmd_latency(a) -> None:
    c = container.read_container(a.input)
    link = _link(a)
    bits = 8 * c.payload_bytes
    print(f"payload_bits={bits} rate_bps={channel.outage_rate(link):.1f} "
          f"t_comm_s={channel.comm_latency(bits, link):.9g}")


def build_parser() -> argparse.ArgumentParser:
    root = _Parser(prog="sczip", description=__doc__.split("\n\n")[0])
    sub = root.add_subparsers(dest="command")

    def cmd(name, fn, help_):
        p = sub.add_parser(name, help=help_)
        p.set_defaults(run=fn)
        return p

    p = cmd("compress", _cmd_compress, "compress an RTF tensor into a .scz container (GPU)")
    p.add_argument("input")
    p.add_argument("--q", type=int, required=True, help="quantisation bit-width")
    p.add_argument("--n", type=int, default=None, help="explicit reshape row count (default: Algorithm 1)")
    p.add_argument("-o", "--output", required=True)
    p.add_argument("--format", type=int, default=container.VERSION, choices=(1, 2),
                   help="1 = reference wire format (default), 2 = interleaved lanes (FORMAT.md)")
    p.add_argument("--block-syms", type=int, default=container.DEFAULT_BLOCK_SYMS)

    p = cmd("decompress", _cmd_decompress, "decode a .scz container (v1 or v2) back to RTF (GPU)")
    p.add_argument("input")
    p.add_argument("-o", "--output", required=True)

    p = cmd("analyze", _cmd_analyze, "print the reshape candidate table (one GPU pass)")
    p.add_argument("input")
    p.add_argument("--q", type=int, required=True)
    p.add_argument("--csv", default=None, help="also write the table as CSV")

    p = cmd("bench", _cmd_bench, "sweep Q values on a synthetic tensor (GPU timings)")
    p.add_argument("--kind", default="relu-laplace", choices=bench.KINDS)
    p.add_argument("--dims", required=True, help="comma-separated, e.g. 128,28,28")
    p.add_argument("--sparsity", type=float, default=0.9)
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--q-list", required=True, help="comma-separated bit-widths")
    p.add_argument("--repetitions", type=int, default=20)
    p.add_argument("--csv", required=True)
    _link_args(p)

    p = cmd("latency", _cmd_latency, "modeled link latency for a container")
    p.add_argument("input")
    _link_args(p)
    return root


def cli_dispatch(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except _UsageError:
        return EXIT_USAGE
    except SystemExit as exc:  # --help
        return int(exc.code or 0)
    if getattr(args, "run", None) is None:
        parser.print_usage(sys.stderr)
        return EXIT_USAGE
    try:
        args.run(args)
    except (ValueError, SczipError, OSError) as exc:
        sys.stderr.write(f"sczip: {exc}\n")
        return EXIT_DATA
    return EXIT_OK


def main() -> None:
    raise SystemExit(cli_dispatch())


if __name__ == "__main__":
    main()
