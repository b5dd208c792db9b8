"""The reference's command line (tools/pathreuse_cli.cpp) over the B200 engine
(paper_2111_06906_b200/cli/pathreuse_cli.cpp): flags, defaults, outputs, exit codes."""
import os
import subprocess

import pytest

from paper_2111_06906_b200 import _lib as L
from paper_2111_06906_b200 import pathreuse as pr
from tests.helpers import counts

CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2111_06906_b200",
                   "pathreuse_cli")
pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="CLI not built (make -C paper_2111_06906_b200)")


def run(*args, **kw):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600, **kw)


def test_help_and_usage_errors(tmp_path):
    r = run("--help")
    assert r.returncode == 0 and "--dump-photons" in r.stdout and "report" in r.stdout
    for bad in (["--mode", "fast"], ["--images", "maybe"], ["--dm", "8x8x64"], ["--dm", "8xx8x64x64"],
                ["--paths", "many"], ["--bogus", "1"], ["report"], ["--frames"]):
        r = run(*bad, "--out", str(tmp_path / "o"))
        assert r.returncode == 2, (bad, r.stdout, r.stderr)
    r = run("--scene", str(tmp_path / "missing.json"), "--out", str(tmp_path / "o"))
    assert r.returncode == 1 and "scene error" in r.stderr


def test_report_subcommand(tmp_path):
    rows = []
    for mode in (0, 1):
        for f in range(2):
            s = L.FrameStats()
            s.frame, s.mode, s.rays_traced, s.rays_reused = f, mode, 1000 - 300 * mode + f, 300 * mode
            rows.append(s)
    pr.write_stats_csv(rows[:2], str(tmp_path / "a.csv"))
    pr.write_stats_csv(rows[2:], str(tmp_path / "b.csv"))
    r = run("report", str(tmp_path / "a.csv"), str(tmp_path / "b.csv"))
    assert r.returncode == 0 and r.stdout == pr.reuse_report(rows)
    r = run("report", str(tmp_path / "b.csv"))  # no baseline rows
    assert r.returncode == 1 and "no baseline" in r.stderr


@pytest.mark.gpu
def test_run_matches_reference(tmp_path):
    from oracle import ref

    out = tmp_path / "run"
    r = run("--scene", "builtin:moving-cube", "--mode", "error", "--paths", "3000", "--bounces", "5",
            "--dm", "2x2x8x8", "--frames", "3", "--seed", "4", "--out", str(out),
            "--dump-photons", str(tmp_path / "final.phm"))
    assert r.returncode == 0, r.stderr
    assert len(r.stdout.splitlines()) == 3
    got = pr.read_stats_csv(str(out / "stats.csv"))
    eng = ref.RefEngine(ref.RefScene.builtin("moving-cube"),
                        pr.make_config("error", paths=3000, bounces=5, dm=[2, 2, 8, 8], seed=4))
    want = [eng.run_frame() for _ in range(3)]
    assert [counts(g) for g in got] == [counts(w) for w in want]
    eng.write_photon_dump(str(tmp_path / "ref.phm"))
    assert (tmp_path / "final.phm").read_bytes() == (tmp_path / "ref.phm").read_bytes()
    for f in range(3):
        assert (out / pr.frame_image_name(f)).stat().st_size > 0
    assert (out / "config.json").exists()
