"""Golden outputs of the REFERENCE command line (unimul.cli) for the CLI parity tests.

Run in the build container (where /root/reference exists):

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli/<name>.cfg (the config files), <name>.ops and
<name>.ir (the reference's `dump-ops` / `dump-ir` stdout) and sweep.csv
(the reference's `sweep` CSV for a small sweep file).  Imports the reference
from /root/reference/pkg/src, read-only.
"""

import contextlib
import io
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from unimul import cli, kernels  # noqa: E402

kernels.gemm_accumulate = kernels.gemm_accumulate_numpy
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")

CONFIGS = {
    "cfg1_c": "m = 1024\nn = 1024\nk = 1024\np = 4\n",
    "cfg1_a": "m = 1024\nn = 1024\nk = 1024\np = 4\nstationarity = a\n",
    "mis_b": "m = 40\nn = 36\nk = 52\np = 6\na_part = misaligned\nb_part = col\nc_part = row\nstationarity = b\n",
    "rep_cost": ("m = 96\nn = 64\nk = 128\np = 8\na_part = 2d\nb_part = 2d\nc_part = 2d\nc_a = 2\nc_b = 2\n"
                 "c_c = 2\nexecution = ir:cost\n"),
    "cyc_auto": ("m = 48\nn = 40\nk = 64\np = 4\na_part = custom:8:8:2:2:cyclic\nb_part = row\n"
                 "c_part = custom:16:8\nstationarity = auto\n"),
    "twolevel": ("m = 64\nn = 64\nk = 64\np = 8\ntopology = twolevel\ngroup_size = 4\ninter_bandwidth = 1e8\n"
                 "execution = ir:greedy\nc_part = row\n"),
}
SWEEP = ("# small acceptance-style sweep\nm = 24, 40\nn = 32\nk = 48\np = 4\na_part = row, 2d\n"
         "b_part = col\nc_part = 2d, misaligned\nstationarity = a, c\nc_c = 1, 2\n")


def capture(fn, *args):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = fn(*args)
    return rc, buf.getvalue()


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, text in CONFIGS.items():
        path = os.path.join(OUT, name + ".cfg")
        with open(path, "w") as f:
            f.write(text)
        for cmd, ext in (("dump-ops", "ops"), ("dump-ir", "ir")):
            rc, out = capture(cli.main, [cmd, path])
            assert rc == 0
            with open(os.path.join(OUT, f"{name}.{ext}"), "w") as f:
                f.write(out)
    sp = os.path.join(OUT, "sweep.sweep")
    with open(sp, "w") as f:
        f.write(SWEEP)
    rc, out = capture(cli.main, ["sweep", sp])
    with open(os.path.join(OUT, "sweep.csv"), "w") as f:
        f.write(out)
    print("wrote", sorted(os.listdir(OUT)), "sweep rc", rc)


if __name__ == "__main__":
    main()
