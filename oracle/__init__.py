"""TEST INFRASTRUCTURE — the checkers of the dock-and-score path.

* ``oracle.ref``   — ctypes bridge to the UNMODIFIED reference library compiled
                     from /root/reference (oracle/_ref/libvsref.so).
* ``oracle.sweep`` — ctypes bridge to the C restatement of sweep-v1
                     (oracle/_ref/libvsoracle.so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(paper_2304_09953_b200) never does.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libvsref.so")
ORACLE_SO = os.path.join(HERE, "_ref", "libvsoracle.so")


def build(ref: bool = True) -> None:
    """Build the oracle (always) and the reference library (when the
    reference tree is present; on the GPU box the prebuilt .so travels)."""
    subprocess.run(["make", "-C", HERE, "oracle"], check=True, stdout=subprocess.DEVNULL)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, stdout=subprocess.DEVNULL)
        # the reference's own dock / batcher unit tests, compiled against the
        # drop-in headers and library (oracle/build_ref_tests.sh)
        subprocess.run(["bash", os.path.join(HERE, "build_ref_tests.sh")], check=True,
                       stdout=subprocess.DEVNULL)
