"""Heat-map files: the analyzer's CSV + region
configuration ("recorded in CSV files", "stored in configuration
files"; formats of S:334) and the run-compressed table of Fig. 4.  Host-side
formatting of what libthermo computed (thermo_query_heatmap / _runs); no
heat-map arithmetic happens here.
"""
from __future__ import annotations

import io

import numpy as np

SPACES = {0: "global", 1: "shared", 2: "local"}
HEAT_HEADER = "space,region_id,sector_tag,w0,w1,w2,w3,w4,w5,w6,w7,sector"
CONFIG_HEADER = "region_id,label,space,base,length,start_tag,end_tag"


def heat_csv(objects, rows_of) -> str:
    """One row per touched sector (sector temperature > 0), objects in the given
    order.  objects: [(base, len, space, id[, label])]; rows_of(id) -> [S, 9]
    (8 word temperatures, then the sector's)."""
    out = io.StringIO()
    out.write(HEAT_HEADER + "\n")
    for o in objects:
        base, space, oid = int(o[0]), int(o[2]), int(o[3])
        rows = np.asarray(rows_of(oid)).reshape(-1, 9)
        for s in np.nonzero(rows[:, 8])[0]:
            vals = ",".join(str(int(v)) for v in rows[s])
            out.write(f"{SPACES[space]},{oid},{(base >> 5) + int(s)},{vals}\n")
    return out.getvalue()


def parse_heat_csv(text: str) -> dict:
    """{(region_id, sector_tag): 9 temperatures} from heat_csv's output."""
    lines = text.strip().split("\n")
    assert lines[0] == HEAT_HEADER
    table = {}
    for ln in lines[1:]:
        f = ln.split(",")
        table[(int(f[1]), int(f[2]))] = [int(x) for x in f[3:]]
    return table


def config_csv(objects) -> str:
    out = io.StringIO()
    out.write(CONFIG_HEADER + "\n")
    for o in objects:
        base, ln, space, oid = (int(x) for x in o[:4])
        label = o[4] if len(o) > 4 else f"region{oid}"
        out.write(f"{oid},{label},{SPACES[space]},{base},{ln},{base >> 5},{(base + ln - 1) >> 5}\n")
    return out.getvalue()


def expand_runs(start, count, temps) -> np.ndarray:
    """Dense rows from a run-compressed table (the inverse of thermo_query_runs)."""
    return np.repeat(np.asarray(temps).reshape(-1, 9), np.asarray(count).astype(np.int64), axis=0)
