"""The tuning cache through the C ABI (dfk_cache_store / dfk_cache_lookup),
restating the reference's cache tests (proj/tests/test_tuner.cpp: "cache
round-trip is exact, misses are clean", "cache file is human-readable and
versioned", "corrupt and future-version cache files are rejected", "cache
survives concurrent writers and readers").  Host-only: runs without a GPU."""
import json
import multiprocessing as mp
import os
import threading

import pytest

from paper_2602_11808_b200 import runtime as rt


def entry(b, dm, df, fp, chosen, results=()):
    return {"shape": {"batch": b, "d_model": dm, "d_ff": df}, "fingerprint": fp,
            "chosen": chosen, "created_at": "2026-08-09T00:00:00Z", "results": list(results)}


def test_round_trip_is_exact_and_misses_are_clean(tmp_path):
    path = str(tmp_path / "c.json")
    e = entry(2, 4, 8, "gpu-A", "fused_x",
              [{"label": "fused_x", "variant": "fused", "samples_ns": [3, 1, 2],
                "median_ns": 2, "warmup_runs": 1, "measured_runs": 3}])
    rt.cache_store(path, e)
    assert rt.cache_lookup(path, 2, 4, 8, "gpu-A") == e
    assert rt.cache_lookup(path, 2, 4, 8, "gpu-B") is None
    assert rt.cache_lookup(path, 9, 9, 9, "gpu-A") is None
    assert rt.cache_lookup(str(tmp_path / "missing.json"), 2, 4, 8, "gpu-A") is None
    # same key replaced, not duplicated
    e2 = dict(e, chosen="two_kernel")
    rt.cache_store(path, e2)
    assert rt.cache_lookup(path, 2, 4, 8, "gpu-A")["chosen"] == "two_kernel"
    doc = json.load(open(path))
    assert len(doc["entries"]) == 1
    # no temporary files left behind
    assert sorted(os.listdir(tmp_path)) == ["c.json", "c.json.lock"]


def test_file_is_human_readable_and_versioned(tmp_path):
    path = str(tmp_path / "v.json")
    rt.cache_store(path, entry(1, 2, 3, "fp", "four_kernel"))
    text = open(path).read()
    assert "format_version" in text and "four_kernel" in text and "\n  " in text


def test_corrupt_and_future_version_files_are_rejected(tmp_path):
    bad = tmp_path / "corrupt.json"
    bad.write_text('{"format_version": 1, "entries": [ {"shap')
    with pytest.raises(rt.CacheError):
        rt.cache_lookup(str(bad), 1, 2, 3, "fp")
    with pytest.raises(rt.CacheError):  # a store must not clobber it either
        rt.cache_store(str(bad), entry(1, 2, 3, "fp", "x"))
    fut = tmp_path / "future.json"
    fut.write_text('{"format_version": 99, "entries": []}')
    with pytest.raises(rt.CacheError, match="version"):
        rt.cache_lookup(str(fut), 1, 2, 3, "fp")
    empty = tmp_path / "empty.json"
    empty.write_text("")
    assert rt.cache_lookup(str(empty), 1, 2, 3, "fp") is None


def test_malformed_new_entry_is_rejected(tmp_path):
    with pytest.raises(rt.CacheError):
        rt.cache_store(str(tmp_path / "m.json"), {"fingerprint": "fp"})


def _writer(path, t, rounds):
    for r in range(rounds):
        rt.cache_store(path, entry(t + 1, 4, 8, "fp", f"fused_round_{r}"))
        rt.cache_lookup(path, t + 1, 4, 8, "fp")


def test_concurrent_writers_threads_and_processes(tmp_path):
    path = str(tmp_path / "cc.json")
    ths = [threading.Thread(target=_writer, args=(path, t, 10)) for t in range(4)]
    procs = [mp.get_context("spawn").Process(target=_writer, args=(path, 4 + t, 10))
             for t in range(3)]
    for x in ths + procs:
        x.start()
    for x in ths + procs:
        x.join()
    assert all(p.exitcode == 0 for p in procs)
    for t in range(7):
        assert rt.cache_lookup(path, t + 1, 4, 8, "fp")["chosen"] == "fused_round_9"
