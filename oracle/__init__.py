"""CPU checkers for the DCO hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package. Two checkers live here:

  oracle.ref   — ctypes access to the UNMODIFIED reference library
                 (/root/reference/proj/src built by oracle/Makefile into
                 oracle/_ref/libdco_ref.so; the .so travels to the GPU box).
  oracle.port  — the C restatement dco_oracle.c (oracle/_lib/libdco_oracle.so),
                 pinned against oracle.ref by tests/test_oracle_port.py.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libdco_ref.so")
PORT_LIB = os.path.join(HERE, "_lib", "libdco_oracle.so")
REFERENCE_SRC = "/root/reference/proj"


def build(quiet=True):
    """Builds oracle/_ref (only where /root/reference exists) and oracle/_lib."""
    import subprocess

    targets = ["port"]
    if os.path.isdir(REFERENCE_SRC):
        targets.insert(0, "ref")
    for t in targets:
        r = subprocess.run(["make", "-s", "-j8", "-C", HERE, t], capture_output=quiet, text=True)
        if r.returncode != 0:
            raise RuntimeError("oracle build (%s) failed:\n%s\n%s" % (t, r.stdout, r.stderr))
