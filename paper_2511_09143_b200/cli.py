"""Command line: `bootstrap-check` (drop-in) and `select` (new).

`bootstrap-check --peers FILE [--legacy]` follows the reference
`pkg/src/migsim/cli.py:151-162`: load JSONL peers, discover (MIG-aware unless
--legacy), build the topology, print labels and the mig_list.  Exit codes
follow cli.py:45-49, 208-225: 0 ok, 2 invalid input (ValueError), 5
bootstrap failure (DuplicateDeviceError / MalformedLabelError), 1 any other
package error.

`select --gpus G --size N` prints the FM rank order (`fm_select` on an idle
cluster) as JSON: what the local launcher binds rank r to.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from .commsim import build_topology, discover_peers, load_peers_jsonl
from .errors import DuplicateDeviceError, MalformedLabelError, MigSimError
from .scheduler import fm_select, make_cluster
from .workload import Job

EXIT_INVALID_CONFIG = 2
EXIT_BOOTSTRAP = 5


def cmd_bootstrap_check(args: argparse.Namespace) -> int:
    comm = discover_peers(load_peers_jsonl(Path(args.peers).read_bytes()),
                          mig_aware=not args.legacy)
    topo = build_topology(comm)
    print(f"communicator of {comm.size} ranks")
    for node in topo.nodes:
        note = "" if node.label == node.canonical else f" (canonical {node.canonical})"
        print(f"  rank {node.rank}: {node.label}{note}")
    print("mig_list:")
    for bus, count in topo.mig_list:
        print(f"  {bus}: {count}")
    return 0


def cmd_select(args: argparse.Namespace) -> int:
    d = fm_select(Job(0, "train", args.size, 0.0, 0.0), make_cluster("FM", args.gpus))
    if d is None:
        print(json.dumps({"job_id": 0, "instances": None}))
        return 0
    print(json.dumps({"job_id": d.job_id, "transport": d.transport_class,
                      "instances": d.instances, "profiles": d.profiles}))
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="flexshm", description=__doc__.splitlines()[0])
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bootstrap-check", help="validate a peer file and print topology")
    p.add_argument("--peers", required=True, help="peer records (JSON lines)")
    p.add_argument("--legacy", action="store_true", help="bus-id-only duplicate detection")
    p.set_defaults(func=cmd_bootstrap_check)
    p = sub.add_parser("select", help="print the FM rank order for a job")
    p.add_argument("--gpus", type=int, required=True)
    p.add_argument("--size", type=int, required=True)
    p.set_defaults(func=cmd_select)
    return parser


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INVALID_CONFIG
    except (DuplicateDeviceError, MalformedLabelError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_BOOTSTRAP
    except MigSimError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
