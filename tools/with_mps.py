"""Run a command as a client of a private MPS daemon: python tools/with_mps.py CMD..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_09143_b200.launcher import MpsDaemon  # noqa: E402

d = MpsDaemon(f"tool-{os.getpid()}")
if not d.start():
    sys.exit("MPS daemon failed to start")
try:
    rc = subprocess.call(sys.argv[1:], env={**os.environ, **d.env})
finally:
    d.stop()
sys.exit(rc)
