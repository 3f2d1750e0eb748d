"""Drop-in boundary from C++: a probe written against the reference's API names
(include/dwdp.hpp adapter) links libdwdp.so and reproduces the reference."""
import os
import subprocess

import pytest

from conftest import ROOT, load_golden


@pytest.fixture(scope="module")
def probe(tmp_path_factory):
    from paper_2604_01621_b200._lib import LIB_PATH, lib
    lib()
    exe = str(tmp_path_factory.mktemp("hpp") / "hpp_probe")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "hpp_probe.cpp"), LIB_PATH,
                        f"-Wl,-rpath,{os.path.dirname(LIB_PATH)}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    return out.splitlines()


def test_hpp_placement_matches_reference(probe):
    golden = {(c["E"], c["N"], c["extra"]): c for c in load_golden("ref_placement.json")}
    for line in probe:
        if not line.startswith("P "):
            continue
        parts = line.split()
        E, N, x, c, red = map(int, parts[1:6])
        g = golden[(E, N, x)]
        assert (c, red) == (g["local_count"], g["redundancy"])
        fetch = [tuple(map(int, p.split(":"))) for p in parts[6:]]
        assert fetch == [tuple(f) for fl in g["fetch"] for f in fl]


def test_hpp_copy_plan_errors_and_routing(probe):
    c = [ln for ln in probe if ln.startswith("C ")][0].split()[1:]
    assert c == ["1,0,2", "2,0,2", "1,2,2", "2,2,2", "1,4,1", "2,4,1"]  # test_copyplan.cpp:61-73
    assert "E ConfigError" in probe                                      # test_placement.cpp:106-108
    r = [ln for ln in probe if ln.startswith("R ")][0].split()[1:]
    golden = [c for c in load_golden("ref_workload.json")["route"]
              if (c["tokens"], c["E"], c["k"], c["skew"], c["seed"]) == (100, 16, 2, 1.2, 1)][0]
    assert list(map(int, r)) == golden["counts"]
