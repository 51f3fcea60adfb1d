"""Heat-map files: CSV/config formats and the
run-table round trip, on host data (the GPU query itself is in the -m gpu
parity tests)."""
import numpy as np

from paper_2507_18729_b200.export import config_csv, expand_runs, heat_csv, parse_heat_csv


def test_fig3b_row_and_round_trip():
    # Fig. 3(b): 8 warps each on a different word of one sector (S:459 example row)
    objects = [(0x0, 64, 0, 1, "x")]
    rows = np.zeros((2, 9), dtype=np.uint32)
    rows[0] = [1] * 8 + [8]
    csv = heat_csv(objects, lambda oid: rows)
    assert csv.split("\n")[1] == "global,1,0,1,1,1,1,1,1,1,1,8"
    assert parse_heat_csv(csv) == {(1, 0): [1] * 8 + [8]}
    assert heat_csv(objects, lambda oid: np.zeros((2, 9), np.uint32)).strip().count("\n") == 0  # header only


def test_config_and_runs():
    objects = [(0x7F0000000000, 4096, 0, 3, "A"), (0x2000, 100, 1, 4, "s")]
    cfg = config_csv(objects).strip().split("\n")
    assert cfg[1] == f"3,A,global,{0x7F0000000000},4096,{0x7F0000000000 >> 5},{(0x7F0000000000 + 4095) >> 5}"
    rng = np.random.default_rng(1)
    dense = rng.integers(0, 3, (50, 9)).astype(np.uint32)
    dense[10:30] = dense[10]
    # runs of the dense rows, computed here by a plain loop, expand back exactly
    st, ct, tp = [], [], []
    for s in range(len(dense)):
        if s and (dense[s] == dense[s - 1]).all():
            ct[-1] += 1
        else:
            st.append(s); ct.append(1); tp.append(dense[s])
    assert np.array_equal(expand_runs(st, ct, tp), dense)
