"""Copy the reference acceptance suite's data tables (Ghia, Ghia & Shin 1982,
Re = 100 lid-driven cavity centreline profiles: proj/data/ghia_re100_*.dat)
into tests/golden/acceptance_data/, so the acceptance binary built here
(oracle/Makefile, target dropin-acceptance) finds them on the GPU box, where
/root/reference does not exist. Run where the reference tree is present."""
import os
import shutil

SRC = "/root/reference/proj/data"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "acceptance_data")

if __name__ == "__main__":
    os.makedirs(DST, exist_ok=True)
    for name in ("ghia_re100_u.dat", "ghia_re100_v.dat"):
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
        print("wrote", os.path.join(DST, name))
