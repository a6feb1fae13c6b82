"""The walk's exact-division claim (siddon_walk.cuh div_rn): one multiply by
RN(1/d) plus one Markstein FMA correction equals IEEE division, so crossing
parameters are bit-identical to the reference's (o + k sp - s)/d."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def test_markstein_division_matches_ieee(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = tmp_path / "mk"
    subprocess.run([cc, "-O2", "-ffp-contract=off", os.path.join(HERE, "native", "markstein_check.c"),
                    "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe), "4000000"], capture_output=True, text=True, check=True).stdout
    assert int(out.strip()) == 0
