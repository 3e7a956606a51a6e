"""Freeze reference outputs as test fixtures (run in the build container).

Inputs come ONLY from the reference itself: oracle/_ref/ref_driver is the
reference's own src/*.cpp compiled in place by oracle/Makefile.  Outputs:

  tests/golden/<name>.json        the reference's 5 byte-frozen goldens, as
                                  re-emitted by its serializer (byte-identical to
                                  /root/reference/proj/tests/data/<name>.json)
  tests/golden/schedule_grid.json.gz
                                  one record per (scheme, P, B, W, costs):
                                  sha256 of the canonical action streams, makespan,
                                  bubble, memory peaks/weights, message counts, and
                                  the full streams + trace for small configs.

  tests/golden/gantt/<name>.{csv,svg}
                                  the reference's trace_to_gantt of each golden's
                                  simulated trace (src/gantt.cpp:91-95)

Usage:  make -C oracle && python tests/golden/make_golden.py
"""
import gzip
import hashlib
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
REF_DATA = "/root/reference/proj/tests/data"

GOLDENS = [("gpipe-p4-b4", "gpipe", 4, 4, 1), ("dapple-p4-b4", "dapple", 4, 4, 1),
           ("chimera-p4-b4", "chimera", 4, 4, 1), ("hanayo-p4-b4-w1", "hanayo", 4, 4, 1),
           ("hanayo-p4-b4-w2", "hanayo", 4, 4, 2)]

COSTS = [(1.0, 2.0, 0.0), (1.0, 2.0, 0.05), (1.0, 3.0, 0.0), (1.0, 2.0, 0.25), (0.7, 1.3, 0.1)]


def canonical(actions):
    return "\n".join(";".join(",".join(str(x) for x in a) for a in dev) for dev in actions)


def grid():
    seen = set()
    for P in (1, 2, 3, 4, 8):
        for W in (1, 2, 3, 4):
            for mult in (1, 2, 3, 8):
                B = P * mult
                if B > 64 or (P == 8 and W == 4 and mult == 8):
                    continue
                for ci, cost in enumerate(COSTS):
                    if ci >= 2 and (P not in (4, 8) or mult > 2):
                        continue
                    key = ("hanayo", P, B, W, cost)
                    if key not in seen:
                        seen.add(key)
                        yield key
    for scheme in ("gpipe", "dapple", "chimera", "chimera-wave"):
        for P in (2, 4, 8):
            for B in (P, 2 * P):
                W_list = (1, 2) if scheme == "chimera-wave" else (1,)
                for W in W_list:
                    for cost in COSTS[:2]:
                        yield (scheme, P, B, W, cost)


def run(*args):
    return subprocess.run([DRIVER, *map(str, args)], check=True, capture_output=True, text=True).stdout


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build the oracle first: make -C oracle")
    for name, scheme, P, B, W in GOLDENS:
        text = run("json", scheme, P, B, W, 1, 1, 2, 0)
        ref_path = os.path.join(REF_DATA, name + ".json")
        if os.path.exists(ref_path):
            assert text == open(ref_path).read(), f"{name}: ref_driver output differs from the stored golden"
        with open(os.path.join(HERE, name + ".json"), "w") as f:
            f.write(text)
    records = []
    for scheme, P, B, W, (tf, tb, tc) in grid():
        d = json.loads(run("dump", scheme, P, B, W, 1, tf, tb, tc))
        n_actions = sum(len(x) for x in d["actions"])
        kinds = [0] * 6
        for dev in d["actions"]:
            for a in dev:
                kinds[a[0]] += 1
        rec = {"scheme": scheme, "P": P, "B": B, "W": W, "cost": [tf, tb, tc],
               "sha256": hashlib.sha256(canonical(d["actions"]).encode()).hexdigest(),
               "makespan": d["makespan"], "bubble": d["bubble"], "peaks": d["peaks"],
               "weights": d["weights"], "kind_counts": kinds,
               "n_comm_events": len(d["comm_events"])}
        if scheme == "hanayo" and P > 1:
            rec["eq1"] = float(run("eq1", P, W, tf, tb, tc))
        if n_actions <= 700:
            rec["actions"] = d["actions"]
            rec["intervals"] = d["intervals"]
            rec["comm_events"] = d["comm_events"]
        records.append(rec)
    with gzip.open(os.path.join(HERE, "schedule_grid.json.gz"), "wt") as f:
        json.dump(records, f, separators=(",", ":"))
    print(f"wrote {len(records)} grid records")


def gantt():
    os.makedirs(os.path.join(HERE, "gantt"), exist_ok=True)
    for name, *_ in GOLDENS:
        for fmt in ("csv", "svg"):
            out = subprocess.run([DRIVER, "gantt", os.path.join(HERE, name + ".json"), fmt], check=True,
                                 capture_output=True, text=True).stdout
            with open(os.path.join(HERE, "gantt", f"{name}.{fmt}"), "w") as f:
                f.write(out)
    print(f"wrote gantt fixtures for {len(GOLDENS)} goldens")


if __name__ == "__main__":
    if sys.argv[1:] == ["gantt"]:
        gantt()
    else:
        main()
        gantt()
