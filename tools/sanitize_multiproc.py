#!/usr/bin/env python3
"""compute-sanitizer on the one-rank-per-process path: two processes on
cuda:0, each under its own `compute-sanitizer --tool <tool>`, running the
epoch-parity LL worker of tests/test_gpu_ll_parity.py (LL allgather /
alltoall / allreduce with parity slot sets, broadcast with the entry
handshake; back-to-back launches, no barriers) with IPC handles.
usage: python tools/sanitize_multiproc.py memcheck|synccheck [launches]"""
import os
import socket
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_ll_parity import WORKER  # noqa: E402


def main():
    tool = sys.argv[1] if len(sys.argv) > 1 else "memcheck"
    n = sys.argv[2] if len(sys.argv) > 2 else "6"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    d = tempfile.mkdtemp()
    script = os.path.join(d, "w.py")
    with open(script, "w") as f:
        f.write(WORKER.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"), port=port))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen(["compute-sanitizer", "--tool", tool, "--print-limit", "20", sys.executable, script,
                               str(r), "2", "ipc", n], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                              env=env) for r in range(2)]
    rc = 0
    for r, p in enumerate(procs):
        out, _ = p.communicate(timeout=1800)
        print(f"===== rank {r} (rc {p.returncode})\n{out}", flush=True)
        rc |= p.returncode
    sys.exit(rc)


if __name__ == "__main__":
    main()
