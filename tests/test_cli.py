"""CLI parity (reference cli.py / tests/test_cli.py): checkpoint text, row formats, resume
pruning and config errors on CPU; full runs, kill-and-resume and the self-test on the GPU."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

from paper_2506_01099_b200 import cli


def run_cli(*args, env=None):
    return subprocess.run([sys.executable, "-m", "paper_2506_01099_b200", *args], capture_output=True, text=True,
                          cwd=ROOT, env=env)


def csv_of(rows):
    return cli.CSV_HEADER + "\n" + "".join(f"{k},{m},{n},{a},{b}\n" for k, m, n, a, b in rows)


# ---------------------------------------------------------------- CPU ----------------------
def test_checkpoint_text_is_bit_exact(tmp_path):
    ck = cli.Progress(5000, 300, 7)
    assert ck.text() == "benelux-checkpoint v1\nlimit=5000\nchunk_size=300\nnext_chunk=7\n"
    path = str(tmp_path / "ck")
    ck.save(path)
    assert cli.Progress.load(path) == ck
    for bad in ("", "benelux-checkpoint v2\nlimit=1\nchunk_size=3\nnext_chunk=0\n",
                "benelux-checkpoint v1\nlimit=x\nchunk_size=3\nnext_chunk=0\n",
                "benelux-checkpoint v1\nlimit=1\nchunk_size=3\nnext_chunk=0\nextra\n"):
        with pytest.raises(ValueError):
            cli.Progress.from_text(bad)


def test_row_formats_and_torn_tail(tmp_path):
    import paper_2506_01099_b200 as bp

    p = bp.BeneluxPair(75, 1215, bp.Kind.FIRST, 15, 38)
    csv, jsonl = cli.RowFormat("csv"), cli.RowFormat("jsonl")
    assert csv.encode(cli.pair_row(p)) == "1,75,1215,15,38\n"
    assert jsonl.encode(cli.pair_row(p)) == '{"kind": 1, "m": 75, "n": 1215, "rad_m": 15, "rad_m1": 38}\n'
    path = tmp_path / "o.csv"
    path.write_text(cli.CSV_HEADER + "\n1,75,1215,15,38\n2,35,43")
    assert csv.read(str(path)) == [(1, 75, 1215, 15, 38)]
    jpath = tmp_path / "o.jsonl"
    jpath.write_text(jsonl.encode((1, 75, 1215, 15, 38)) + '{"kind": 2, "m"')
    assert jsonl.read(str(jpath)) == [(1, 75, 1215, 15, 38)]
    assert cli.canonical_csv([(2, 3, 8, 3, 2), (1, 2, 8, 2, 3)]) == cli.CSV_HEADER + "\n1,2,8,2,3\n2,3,8,3,2\n"


def test_prune_for_resume(tmp_path):
    path = tmp_path / "o.csv"
    path.write_text(cli.CSV_HEADER + "\n2,2,3,2,3\n1,2,8,2,3\n1,75,1215,15,38\n")
    cli.keep_rows_through(str(path), cli.RowFormat("csv"), 100)
    assert path.read_text() == cli.CSV_HEADER + "\n2,2,3,2,3\n1,2,8,2,3\n"


@pytest.mark.parametrize("args", [
    ["--limit", "2", "--output", "x.csv"],
    ["--limit", "100", "--output", "x.csv", "--algo", "chunked", "--chunk-size", "2"],
    ["--limit", "100", "--output", "x.csv", "--resume"],
    ["--limit", "100", "--output", "x.csv", "--algo", "sort", "--resume", "--checkpoint", "c"],
    ["--limit", "100", "--output", "x.csv", "--threads", "0"],
    ["--limit", "100", "--output", "x.csv", "--algo", "table", "--chunk-size", "1"],
])
def test_config_errors_exit_2(args, tmp_path):
    args = [a if a != "x.csv" else str(tmp_path / "x.csv") for a in args]
    assert cli.main(args) == 2


def test_missing_arguments_exit_2():
    assert cli.main(["--output", "x"]) == 2
    assert cli.main(["--limit", "10"]) == 2


# ---------------------------------------------------------------- GPU ----------------------
@pytest.mark.gpu
def test_sort_run_rows(tmp_path, golden):
    out = tmp_path / "s.csv"
    r = run_cli("--limit", str(2**20), "--output", str(out))
    assert r.returncode == 0, r.stderr
    assert out.read_text() == csv_of(golden["find_pairs_sorted"]["1048576"])


@pytest.mark.gpu
def test_chunked_run_bytes_and_formats(tmp_path, golden):
    out = tmp_path / "c.csv"
    r = run_cli("--limit", str(2**20), "--algo", "chunked", "--chunk-size", "4096", "--output", str(out))
    assert r.returncode == 0, r.stderr
    assert out.read_text() == csv_of(golden["run_full_chunked"]["1048576_4096"])
    js = tmp_path / "c.jsonl"
    assert run_cli("--limit", str(2**20), "--algo", "chunked", "--chunk-size", "4096", "--format", "jsonl",
                   "--output", str(js)).returncode == 0
    assert cli.canonical_file(str(js), "jsonl") == cli.canonical_file(str(out), "csv")
    tb = tmp_path / "t.csv"  # the paper's Algorithm 3: same bytes as the chunked run
    assert run_cli("--limit", str(2**20), "--algo", "table", "--chunk-size", "65536",
                   "--output", str(tb)).returncode == 0
    assert tb.read_text() == csv_of(golden["run_full_chunked"]["1048576_65536"])


@pytest.mark.gpu
def test_kill_and_resume_is_byte_identical(tmp_path):
    full = tmp_path / "full.csv"
    assert run_cli("--limit", "4194304", "--algo", "chunked", "--chunk-size", "16384",
                   "--output", str(full)).returncode == 0
    for abort_at in (0, 37, 200):
        out, ck = tmp_path / f"r{abort_at}.csv", tmp_path / f"r{abort_at}.ck"
        r = run_cli("--limit", "4194304", "--algo", "chunked", "--chunk-size", "16384", "--output", str(out),
                    "--checkpoint", str(ck), "--abort-after-chunk", str(abort_at))
        assert r.returncode == 3
        assert cli.Progress.load(str(ck)).next_chunk == abort_at + 1
        r = run_cli("--limit", "4194304", "--algo", "chunked", "--chunk-size", "16384", "--output", str(out),
                    "--checkpoint", str(ck), "--resume")
        assert r.returncode == 0, r.stderr
        assert out.read_bytes() == full.read_bytes()


@pytest.mark.gpu
def test_checkpoint_mismatch_exit_1(tmp_path):
    out, ck = tmp_path / "o.csv", tmp_path / "o.ck"
    cli.Progress(5000, 300, 2).save(str(ck))
    r = run_cli("--limit", "6000", "--algo", "chunked", "--chunk-size", "300", "--output", str(out),
                "--checkpoint", str(ck), "--resume")
    assert r.returncode == 1 and "checkpoint" in r.stderr


@pytest.mark.gpu
def test_resume_refuses_another_kind(tmp_path, golden):
    """A --kind run records its kind beside the checkpoint; resuming it with another kind is a
    checkpoint mismatch (exit 1), resuming with the same kind completes the filtered file."""
    out, ck = tmp_path / "k.csv", tmp_path / "k.ck"
    args = ["--limit", str(2**20), "--algo", "chunked", "--chunk-size", "4096", "--output", str(out),
            "--checkpoint", str(ck)]
    assert run_cli(*args, "--kind", "first", "--abort-after-chunk", "20").returncode == 3
    r = run_cli(*args, "--resume")
    assert r.returncode == 1 and "kind" in r.stderr
    assert run_cli(*args, "--kind", "first", "--resume").returncode == 0
    want = [r for r in golden["run_full_chunked"]["1048576_4096"] if r[0] == 1]
    assert out.read_text() == csv_of(want)


@pytest.mark.gpu
def test_kind_flag(tmp_path, golden):
    out = tmp_path / "k.csv"
    assert run_cli("--limit", str(2**20), "--kind", "second", "--output", str(out)).returncode == 0
    want = [r for r in golden["find_pairs_sorted"]["1048576"] if r[0] == 2]
    assert out.read_text() == csv_of(want)


@pytest.mark.gpu
def test_self_test_passes():
    r = run_cli("--self-test")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "5/5 checks passed" in r.stdout


@pytest.mark.gpu
def test_gpu_brute_force_golden(golden):
    import paper_2506_01099_b200 as bp

    for lim, rows in golden["brute_force"].items():
        got = [[int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1] for p in bp.brute_force_pairs(int(lim))]
        assert got == rows


@pytest.mark.gpu
def test_paper_range_run_with_checkpoints(tmp_path):
    """The paper's full range through the CLI's chunked run at the reference's default chunk
    (2^27: 10,431 chunks, a checkpoint after each): the rows equal Theorem 1 (42 pairs), and a
    resume from the finished checkpoint leaves the file unchanged."""
    from oracle import theorem1

    out, ck = tmp_path / "p.csv", tmp_path / "p.ck"
    args = ["--limit", str(theorem1.COMPLETENESS_BOUND), "--algo", "chunked", "--chunk-size", str(2**27),
            "--output", str(out), "--checkpoint", str(ck)]
    r = run_cli(*args)
    assert r.returncode == 0, r.stderr
    want = theorem1.known_rows(theorem1.COMPLETENESS_BOUND)
    assert cli.canonical_file(str(out), "csv") == cli.canonical_csv(want)
    assert cli.Progress.load(str(ck)).next_chunk == 10431
    before = out.read_bytes()
    assert run_cli(*args, "--resume").returncode == 0
    assert out.read_bytes() == before
