"""The C-ABI library loads without a GPU and exports every symbol
include/ecco_b200.h declares (no compute calls here)."""
import os
import re
import subprocess

import paper_2512_11727_b200 as ecco
from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ecco_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^[ \t]*(?:const\s+)?[\w]+\s*\**\s*(ecco_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    L = ecco.lib()
    declared = declared_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(ecco.EXPORTS) == declared


def test_kernels_are_sm100a_cubins():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ecco.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_product_does_not_link_the_oracle():
    out = subprocess.run(["nm", "-D", ecco.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out and "ref_" not in out
