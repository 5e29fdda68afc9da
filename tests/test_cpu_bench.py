"""bench.py's host-side accounting (no GPU): algorithmic bytes per lattice
update (SURVEY.md §8(d) census rule 2 x arrays x s, and the M schedule's
2 x moments x s), and the porous workload's geometry generator."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2304_06437_b200 import tslb as T  # noqa: E402


def test_census_bytes_per_update():
    # bench.hpp:62-63: D2Q9 120 B, D3Q19 232 B, D3Q27 296 B at fp32 (F1)
    for lat, b in (("d2q9", 120), ("d3q19", 232), ("d3q27", 296)):
        assert bench.step_bytes(T.lattice_of(lat), 1, 4, "f1") == b
    # M: 2 x (1 + D + D(D+1)/2) x s
    assert bench.step_bytes(T.lattice_of("d3q19"), 1, 4, "m") == 80
    assert bench.step_bytes(T.lattice_of("d2q9"), 1, 4, "m") == 48
    assert bench.step_bytes(T.lattice_of("d3q19"), 1, 8, "m") == 160


def test_masked_bytes_add_the_geometry():
    L = T.lattice_of("d3q19")
    plain, masked = bench.kernel_bytes(L, 1, 4), bench.kernel_bytes(L, 1, 4, True)
    assert masked["mstep"] - plain["mstep"] == 4          # u32 solid bits
    assert masked["moments"] - plain["moments"] == 1      # u8 solid mask
    assert masked["streamcoll"] - plain["streamcoll"] == 5  # mask + u32 slow mask


def test_sphere_pack_is_deterministic_and_hits_its_fraction():
    a = bench.sphere_pack((96, 64, 48), 6.0, 0.25, 5)
    b = bench.sphere_pack((96, 64, 48), 6.0, 0.25, 5)
    assert a.dtype == np.uint8 and a.shape == (96 * 64 * 48,)
    assert np.array_equal(a, b)
    assert 0.2 < a.mean() < 0.3
    # periodic: spheres wrap across every face
    s = a.reshape(48, 64, 96)
    assert s[:, :, 0].any() and s[:, :, -1].any() and s[0].any() and s[-1].any()


def test_traffic_captures_match_the_bench_accounting():
    # profiles/traffic.json feeds roofline.traffic: every entry names a
    # committed capture, a bench workload, and the algorithmic bytes that
    # kernel_bytes assigns to the same kernel class
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    t = json.load(open(os.path.join(root, "profiles", "traffic.json")))
    for key, e in t.items():
        if key.startswith("_"):
            continue
        lat, storage, kind = key.split("/")
        masked = kind.endswith("+solid")
        kind = kind.replace("+solid", "")
        assert os.path.exists(os.path.join(root, e["source"].split(" ")[0])), key
        assert e["workloads"] and all(w in bench.WORKLOADS for w in e["workloads"]), key
        L = T.lattice_of(lat)
        comps = 2 if kind.startswith("cg_") else 1
        es = {"f32": 4, "f64": 8, "f16": 2}[storage]
        kb = bench.kernel_bytes(L, comps, es, masked)
        if kind == "cg_streamcoll":
            # box geometries fold the gradient in: phi read instead of grad
            npi = L.dim * (L.dim + 1) // 2
            kb[kind] = (3 + L.dim + npi + 1 + 2 * L.q) * es
        if kind in kb:
            assert kb[kind] == e["algorithmic"], key
        # measured DRAM bytes within 10 % of the algorithmic figure
        assert 0.95 < e["bytes_per_node"] / e["algorithmic"] < 1.1, key


def _run_bench(args, env=None, timeout=300):
    import subprocess
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), *args], capture_output=True,
                          text=True, env=e, timeout=timeout)


def test_gpus_flag_launches_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1); --launch-check reports them over gloo."""
    import json
    r = _run_bench(["--gpus", "2", "--launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["n_gpus"] == 2 and out["ranks"] == [0, 1] and out["pids_distinct"]


def test_relaunch_passes_the_cube_option_through():
    """`--n` is an abbreviation torch.distributed.run's own parser would
    claim (even after the script path): the relaunch passes it as --cube."""
    import json
    r = _run_bench(["--gpus", "2", "--n", "64", "--launch-check"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["n_gpus"] == 2


def test_gpus_flag_must_match_world_size():
    r = _run_bench(["--gpus", "4", "--launch-check"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_strong_scaling_workload_splits_the_fixed_domain():
    w = bench.WORKLOADS["tgv-c5"]
    assert w["dims"] == (2048, 1024, 1024) and w.get("strong")
    for n in (1, 2, 4, 8):
        assert w["dims"][2] % n == 0
