"""Generate the C5 sweep goldens from the pinned C oracle (test infrastructure).

    python tests/golden/make_c5_golden.py full  [workers]   # nb=1024, D=256, seed 0: all 456 calls
    python tests/golden/make_c5_golden.py first [workers]   # reference-semantics answers, sweep grid

The oracle (oracle/pipecut_oracle.c) is pinned to the reference itself by
tests/test_oracle.py (the reference's DP families, known optima, every span of
random and model graphs, the C5 chain goldens made by make_golden.py from
/root/reference).  The reference's own Python needs hours per call at these
sizes, so the goldens come from the oracle, one DP call per worker process
(calls are independent: stages.py:282-291 builds a fresh _Profiler per call,
and the oracle's memo only caches the same deterministic records).

The (n, S, MB) enumeration and the first-feasible-level selection below restate
form_stage (pkg/src/pipecut/stages.py:372-413); `selfcheck()` pins them to the
reference's chain goldens (chains.json) and to the oracle's own orc_form_stage
before anything is written.

Per call the fixture records: the call (S, D, R, MB), its widening level, the
reference's pruned SearchStats.visits of the call (default options), whether a
plan exists, its objective and simulated iteration time as float.hex, and the
plan's stage boundaries and device counts (t_fwd/t_bwd/mem of the stages are
pinned through a digest of their hex strings).
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import cases  # noqa: E402
from oracle.oracle import PC_OK, OracleProblem  # noqa: E402
from paper_2103_16063_b200.flatten import flatten_blockset  # noqa: E402

FULL_POINT = (1024, 256, 0)
FIRST_GRID = [(nb, D, seed) for nb in (256, 1024, 4096) for D in (8, 64, 256)
              for seed in range(5)]


def enumerate_calls(num_nodes, dpn, batch_size, nb):
    """form_stage's candidate loop (stages.py:389-403): widening level n,
    S ascending, MB doubling."""
    out, n, lv = [], 1, 0
    while n <= num_nodes:
        if num_nodes % n == 0:
            D, R = dpn * n, num_nodes // n
            for S in range(dpn * (n - 1) + 1, D + 1):
                if S > nb:
                    continue
                MB = 1
                while MB * R <= batch_size:
                    out.append((lv, (S, D, R, MB)))
                    MB *= 2
            lv += 1
        n *= 2
    return out


def unpruned(nb, call):
    S, D, _, _ = call
    A, B = nb - S + 1, D - S + 1
    return S * (A * (A + 1) // 2) * (B * (B + 1) // 2)


def stage_digest(stages):
    h = hashlib.sha256()
    for (lo, hi, dev, tf, tb, mem) in stages:
        h.update(f"{lo},{hi},{dev},{tf.hex()},{tb.hex()},{mem};".encode())
    return h.hexdigest()[:32]


_OP = {}


def _problem(nb, D, seed):
    key = (nb, D, seed)
    if key not in _OP:
        _OP.clear()
        _OP[key] = OracleProblem(flatten_blockset(cases.c5_blockset(nb, D, jitter_seed=seed)))
    return _OP[key]


def run_call(args):
    (nb, D, seed), call = args
    S, Dc, R, MB = call
    op = _problem(nb, D, seed)
    t0 = time.time()
    rc, stages, obj, visits = op.form_stage_dp(S, Dc, 8 * D, R, MB)
    rec = {"call": list(call), "visits": visits, "feasible": rc == PC_OK,
           "seconds": round(time.time() - t0, 2)}
    if rc == PC_OK:
        it = op.simulate(stages, 8 * D, R, MB)
        rec.update(objective=obj.hex(), iteration_time=it.hex(),
                   bounds=[s[0] for s in stages] + [stages[-1][1]],
                   devices=[s[2] for s in stages], stage_digest=stage_digest(stages))
    return rec


def select(recs, levels):
    """First feasible widening level; within it min by (iteration time,
    objective, MB), first in call order (stages.py:404-413).  Returns
    (index or None, visits, dp_calls) as the reference's SearchStats count them."""
    visits = calls = 0
    i = 0
    while i < len(recs):
        lv = levels[i]
        best = None
        while i < len(recs) and levels[i] == lv:
            r = recs[i]
            visits += r["visits"]
            calls += 1
            if r["feasible"]:
                key = (float.fromhex(r["iteration_time"]), float.fromhex(r["objective"]),
                       r["call"][3])
                if best is None or key < best[0]:
                    best = (key, i)
            i += 1
        if best is not None:
            return best[1], visits, calls
    return None, visits, calls


def run_point(pool, point, first_only):
    nb, D, seed = point
    N, dpn = max(1, D // 8), min(8, D)
    enum = enumerate_calls(N, dpn, 8 * D, nb)
    levels = [lv for lv, _ in enum]
    calls = [c for _, c in enum]
    recs = [None] * len(calls)
    lv = 0
    while lv <= max(levels):
        idx = [i for i in range(len(calls)) if levels[i] == lv] if first_only else \
            list(range(len(calls)))
        idx.sort(key=lambda i: -unpruned(nb, calls[i]))
        for i, r in zip(idx, pool.imap(run_call, [(point, calls[i]) for i in idx])):
            recs[i] = r
        if not first_only or any(recs[i]["feasible"] for i in idx):
            break
        lv += 1
    n_done = sum(r is not None for r in recs)
    done = recs[:n_done]
    assert all(r is not None for r in done)
    win, visits, dp_calls = select(done, levels[:n_done])
    return {"nb": nb, "D": D, "seed": seed, "batch": 8 * D, "nodes": N, "dpn": dpn,
            "answer": None if win is None else dict(done[win], index=win),
            "visits": visits, "dp_calls": dp_calls, "levels": levels[:n_done], "calls": done}


def selfcheck(pool):
    """The parallel per-call path + select() equals the reference's goldens
    (chains.json, made from /root/reference by make_golden.py) on the points
    it holds, and the oracle's own orc_form_stage."""
    with open(os.path.join(HERE, "chains.json")) as fh:
        gold = json.load(fh)
    for key, (nb, D, seed) in (("nb64_D8_seed0", (64, 8, 0)), ("nb32_D16_seed1", (32, 16, 1))):
        doc = run_point(pool, (nb, D, seed), first_only=True)
        want = gold[key]
        a = doc["answer"]
        assert a["objective"] == want["plan"]["objective"], (key, a, want)
        assert a["bounds"] == [s[0] for s in want["plan"]["stages"]] + [want["plan"]["stages"][-1][1]]
        assert a["devices"] == [s[2] for s in want["plan"]["stages"]]
        assert a["call"][2:] == [want["plan"]["replica_factor"], want["plan"]["microbatches"]]
        assert doc["dp_calls"] == want["dp_calls"]
        op = _problem(nb, D, seed)
        rc, plan, visits, calls = op.form_stage(max(1, D // 8), min(8, D), 8 * D)
        assert rc == PC_OK and plan["objective"].hex() == a["objective"]
        assert visits == doc["visits"] and calls == doc["dp_calls"]
    print("selfcheck ok", flush=True)


def dump(name, doc):
    path = os.path.join(HERE, name)
    with open(path + ".tmp", "w") as fh:
        json.dump(doc, fh, separators=(",", ":"), sort_keys=True)
        fh.write("\n")
    os.replace(path + ".tmp", path)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "first"
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else max(1, (os.cpu_count() or 2) - 2)
    with mp.get_context("fork").Pool(workers, maxtasksperchild=8) as pool:
        selfcheck(pool)
        if what == "full":
            t0 = time.time()
            doc = run_point(pool, FULL_POINT, first_only=False)
            doc["generated_seconds"] = round(time.time() - t0)
            dump("c5_full_nb1024_D256_seed0.json", doc)
            print("full done", doc["answer"]["objective"], doc["visits"], flush=True)
        else:
            path = os.path.join(HERE, "c5_first_level.json")
            out = json.load(open(path)) if os.path.exists(path) else {}
            # cheap points first, then seed 0 of every point, then the other seeds
            for point in sorted(FIRST_GRID, key=lambda p: (p[0] == 4096 and p[1] > 8,
                                                           p[2] > 0, p[0], p[1], p[2])):
                key = "nb{}_D{}_seed{}".format(*point)
                if key in out:
                    continue
                t0 = time.time()
                doc = run_point(pool, point, first_only=True)
                doc["generated_seconds"] = round(time.time() - t0)
                out[key] = doc
                dump("c5_first_level.json", out)
                a = doc["answer"]
                print(key, None if a is None else (a["objective"], a["call"]), doc["visits"],
                      doc["dp_calls"], f"{time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
