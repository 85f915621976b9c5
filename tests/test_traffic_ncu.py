"""GPU counterpart of the reference's traffic-model exactness check
(criterion 3, verification.cpp:332-379, and the no-intermediate check
:877-907): ncu's DRAM and SM->L2 write counters of ONE block call vs the
reference's fused single-tile traffic model (traffic.cpp:70-76, 82-94, at
2 B/element), plus a MaterializeIntermediate control -- the unfused
two-kernel layout, whose [A_gate | A_1] round trip must show up in the
write counter.  Skipped when ncu is absent."""
import csv
import io
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum"


def counters(B, variant, dm=4096, df=14336):
    if not os.path.exists(NCU):
        pytest.skip("ncu not available")
    cmd = [NCU, "--profile-from-start", "off", "--metrics", METRICS, "--csv",
           sys.executable, os.path.join(ROOT, "tools", "traffic_check.py"), "--B", str(B),
           "--variant", variant, "--dm", str(dm), "--df", str(df)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout[r.stdout.index('"ID"'):]
    tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0,
           "lts__t_sectors_srcunit_tex_op_write.sum": 0.0}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1}
    for row in csv.DictReader(io.StringIO(lines)):
        name = row["Metric Name"]
        if name in tot:
            v = float(row["Metric Value"].replace(",", ""))
            tot[name] += v * scale.get(row["Metric Unit"], 1)
    return tot


@pytest.mark.parametrize("B", [1, 64])
def test_fused_block_dram_matches_traffic_model(B):
    dm, df = 4096, 14336
    c = counters(B, "fused", dm, df)
    alg = 2 * (3 * dm * df + 2 * B * dm + 2 * B * df)  # traffic.cpp fused model
    dram = c["dram__bytes_read.sum"] + c["dram__bytes_write.sum"]
    assert abs(dram / alg - 1) < 0.03, (dram, alg)
    # SM->L2 stores: A2 (bf16) + the zeroing of Y (fp32; the down partial sums
    # are then red.adds straight into Y -- "direct Y", no workspace, finalize
    # or re-zeroing) + flags / queue words (7.2 KB at B = 1 and 64).  20 KB of slack:
    # ONE materialised intermediate -- A_gate alone in bf16, B x d_ff x 2 B =
    # 28 KB at B = 1, 1.8 MB at B = 64 -- exceeds it.
    writes = c["lts__t_sectors_srcunit_tex_op_write.sum"] * 32
    assert expected_writes(B, dm, df) <= writes <= expected_writes(B, dm, df) + 20480, (
        writes, expected_writes(B, dm, df))


def expected_writes(B, dm, df, sms=148, tail=True):
    """A2 + the zeroing of Y, plus -- at N >= 32, where the default splits the
    stage-1 tiles past the first wave into 3 K parts (the tail split,
    dfk_config.s1_tail) -- the re-zeroing of those tiles' fp32 partial-sum
    workspace by the CTA that finalises each of them."""
    n_pad = -(-B // 16) * 16
    t1 = -(-df // 64)
    rezero = (t1 - sms) * 128 * n_pad * 4 if tail and n_pad >= 32 and t1 > sms else 0
    return 2 * B * df + 4 * B * dm + rezero


def test_materialized_intermediates_trip_the_write_counter():
    """The two-kernel layout writes [A_gate | A_1] (2 x B x d_ff bf16) and
    reads it back: the counter must see at least that much more than the
    fused block (the reference's MaterializeIntermediate mutant)."""
    B, dm, df = 64, 4096, 14336
    # (whole stage-1 tiles: the N >= 32 tail split's workspace re-zeroing is
    # not an intermediate and would eat into the margin)
    fused = counters(B, "fused_notail", dm, df)["lts__t_sectors_srcunit_tex_op_write.sum"] * 32
    two = counters(B, "two", dm, df)["lts__t_sectors_srcunit_tex_op_write.sum"] * 32
    assert two - fused >= 0.9 * 2 * B * df * 2, (two, fused)


@pytest.mark.parametrize("B", [1, 64])
def test_in_kernel_materialize_mutant_trips_the_write_counter(B):
    """Negative control inside the fused kernel itself (dfk_config.mutant = 2:
    the stage-1 epilogue stores SiLU(A_gate) to global memory as fp32 and
    reloads it, same numbers): its B x d_ff x 4 B of extra stores must fail
    the fused bound above and show up in full."""
    dm, df = 4096, 14336
    # (both with whole stage-1 tiles: the mutant lives in the whole-tile epilogue)
    fused = counters(B, "fused_notail", dm, df)["lts__t_sectors_srcunit_tex_op_write.sum"] * 32
    mut = counters(B, "mutant2", dm, df)["lts__t_sectors_srcunit_tex_op_write.sum"] * 32
    expected = expected_writes(B, dm, df, tail=False)
    assert expected <= fused <= expected + 20480, (fused, expected)
    assert mut > expected + 20480, (mut, expected)
    assert mut - fused >= 0.95 * B * df * 4, (mut, fused)
