"""Generate the committed golden vectors from the reference compiled in place.

Run in a container that has /root/reference (oracle/_ref/libxts_ref.so built by
`make -C oracle`):  python -m tests.golden.make_golden
Every array here is produced by the UNMODIFIED reference code path named next
to it; tests compare the product (and the restated oracle) against them.
"""
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

# make_ensemble configs (compression.cpp:115-200)
CONFIGS = {
    "c1": {"dims": [200, 200, 200], "red": [30, 30, 30], "P": 12, "S": 10, "seed": 0x5eed, "kind": 0},
    "rag": {"dims": [67, 45, 23], "red": [7, 5, 3], "P": 3, "S": 2, "seed": 17, "kind": 0},
    "sp": {"dims": [100, 90, 80], "red": [10, 9, 8], "P": 3, "S": 2, "seed": 5, "kind": 1, "s": 4.0},
    "one": {"dims": [8, 8, 8], "red": [3, 3, 3], "P": 2, "S": 1, "seed": 502, "kind": 0},
}


def main():
    import sys
    sys.path.insert(0, str(HERE.parents[1]))
    from oracle.oracle import Reference
    ref = Reference()
    out = {}
    for tag, c in CONFIGS.items():
        ens = ref.make_ensemble(c["dims"], c["red"], c["P"], c["S"], seed=c["seed"], kind=c["kind"],
                                s=c.get("s", 1.0))
        for m in range(3):
            for p, mat in enumerate(ens[m]):
                out[f"ens_{tag}_{m}_{p}"] = mat
    # rng.hpp:26-41 stream and std::log on polar-method inputs
    out["normals_seed12345"] = ref.rng_normal(12345, 4096)
    np.savez_compressed(HERE / "ensembles.npz", **out)

    # compression.cpp:211-213 on a seeded tensor + the "rag" ensemble
    c = CONFIGS["rag"]
    rng = np.random.default_rng(2024)
    t = np.asfortranarray(rng.standard_normal(c["dims"]))
    ens = ref.make_ensemble(c["dims"], c["red"], c["P"], c["S"], seed=c["seed"])
    comp = {"t": t}
    for p in range(c["P"]):
        comp[f"y_{p}"] = ref.comp(t, ens[0][p], ens[1][p], ens[2][p])
    # comp_from_factors (compression.cpp:215-220) on generate() factors (pipeline.cpp:182-220)
    a, b, cc = ref.generate(c["dims"], 4, 1)
    comp["a"], comp["b"], comp["c"] = a, b, cc
    for p in range(c["P"]):
        comp[f"yf_{p}"] = ref.comp_from_factors(a, b, cc, ens[0][p], ens[1][p], ens[2][p])
    np.savez_compressed(HERE / "comp.npz", **comp)

    # full decompose (pipeline.cpp:242-575) on config-1 with S = 10 (S = 20 is ill-posed)
    d = {}
    a, b, cc = ref.generate([200, 200, 200], 10, 1)
    rc, rec, st = ref.decompose((a, b, cc), [200, 200, 200], [30, 30, 30], 10, 12, 10, seed=2)
    assert rc == 0
    d["truth_a"], d["truth_b"], d["truth_c"] = a, b, cc
    d["rec_a"], d["rec_b"], d["rec_c"] = rec
    d["stats"] = st
    rc2, _, _ = ref.decompose((a, b, cc), [200, 200, 200], [30, 30, 30], 10, 12, 20, seed=2)
    d["default_S_status"] = np.array([rc2])
    np.savez_compressed(HERE / "decompose_c1.npz", **d)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
