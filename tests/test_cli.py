"""`alto` CLI on the device path: the reference CLI's
subcommands, JSON report keys and exit codes (pkg/tests/test_cli.py)."""

import json

import numpy as np
import pytest

from conftest import EXAMPLE_COORDS, EXAMPLE_DIMS, EXAMPLE_LINEAR, EXAMPLE_VALUES


@pytest.fixture
def cli():
    import importlib

    return importlib.import_module("paper_2102_10245_b200.cli")


@pytest.fixture
def example_tns(tmp_path):
    lines = ["# dims: " + " ".join(str(d) for d in EXAMPLE_DIMS)]
    for c, v in zip(EXAMPLE_COORDS, EXAMPLE_VALUES):
        lines.append(" ".join(str(x + 1) for x in c) + f" {v}")
    p = tmp_path / "example.tns"
    p.write_text("\n".join(lines) + "\n")
    return str(p)


def run(cli, capsys, argv):
    rc = cli.main(argv)
    out = capsys.readouterr().out
    return rc, json.loads(out) if out.strip() else None


class TestUsage:
    """Argument errors and unreadable inputs (no device work; CPU)."""

    def test_no_subcommand(self, cli):
        with pytest.raises(SystemExit) as exc:
            cli.main([])
        assert exc.value.code == 2

    def test_unknown_strategy(self, cli, example_tns):
        with pytest.raises(SystemExit) as exc:
            cli.main(["mttkrp", example_tns, "--mode", "1", "--strategy", "magic"])
        assert exc.value.code == 2

    def test_missing_file_is_io_error(self, cli, tmp_path):
        assert cli.main(["mttkrp", str(tmp_path / "nope.tns"), "--mode", "1"]) == 3

    def test_malformed_text_is_format_error(self, cli, tmp_path):
        p = tmp_path / "bad.tns"
        p.write_text("1 x 1 1.0\n")
        assert cli.main(["check", str(p), "--mode", "1"]) == 3

    def test_bad_container_is_format_error(self, cli, tmp_path):
        p = tmp_path / "bad.alto"
        p.write_bytes(b"ALTO\x09\x03\x40\x00")
        assert cli.main(["cpd", str(p)]) == 3


@pytest.mark.gpu
class TestDevice:
    def test_convert_round_trip(self, cli, capsys, example_tns, tmp_path):
        import paper_2102_10245_b200 as at

        dst = str(tmp_path / "example.alto")
        rc, rep = run(cli, capsys, ["convert", example_tns, dst])
        assert rc == 0 and rep["direction"] == "text-to-binary"
        assert rep["dims"] == list(EXAMPLE_DIMS) and rep["nnz"] == 6 and rep["width"] == 64
        assert rep["masks"] == ["0xa", "0x34", "0x1"]
        back = at.read_alto(dst)
        assert [int(x) for x in back.indices[:, 0]] == EXAMPLE_LINEAR
        txt = str(tmp_path / "back.tns")
        rc, rep = run(cli, capsys, ["convert", dst, txt])
        assert rc == 0 and rep["direction"] == "binary-to-text"
        with open(example_tns) as f, open(txt) as g:
            assert at.parse_tns(g).isequal(at.parse_tns(f))

    def test_mttkrp_report(self, cli, capsys, example_tns):
        rc, rep = run(cli, capsys, ["mttkrp", example_tns, "--mode", "1", "--rank", "2", "--iters", "3",
                                    "--warmup", "1", "--workers", "2", "--check"])
        assert rc == 0
        assert rep["strategy"] == "atomic" and len(rep["times_s"]) == 3
        assert rep["mean_s"] >= rep["min_s"] >= 0 and rep["throughput_per_s"] > 0
        assert rep["check"]["pass"] is True
        rc, rep = run(cli, capsys, ["mttkrp", example_tns, "--mode", "1", "--iters", "1", "--strategy", "buffered",
                                    "--workers", "1"])
        assert rc == 0 and rep["strategy"] == "buffered"

    def test_mode_and_iteration_errors(self, cli, capsys, example_tns):
        assert cli.main(["mttkrp", example_tns, "--mode", "4"]) == 2
        assert cli.main(["mttkrp", example_tns, "--mode", "0"]) == 2
        assert cli.main(["mttkrp", example_tns, "--mode", "1", "--iters", "0"]) == 2
        assert cli.main(["check", example_tns, "--mode", "9"]) == 2

    def test_workers_env(self, cli, capsys, example_tns, monkeypatch):
        monkeypatch.setenv("ALTOTENSOR_WORKERS", "3")
        rc, rep = run(cli, capsys, ["mttkrp", example_tns, "--mode", "1", "--iters", "1"])
        assert rc == 0 and rep["workers"] == 3 and rep["partitions"] == 3
        rc, rep = run(cli, capsys, ["mttkrp", example_tns, "--mode", "1", "--iters", "1", "--workers", "2"])
        assert rep["workers"] == 2
        monkeypatch.setenv("ALTOTENSOR_WORKERS", "many")
        assert cli.main(["mttkrp", example_tns, "--mode", "1", "--iters", "1"]) == 2

    def test_cpd_json_and_csv(self, cli, capsys, tmp_path):
        import paper_2102_10245_b200 as at

        t = at.random_tensor((10, 9, 8), 300, seed=2)
        src = tmp_path / "t.tns"
        with open(src, "w") as f:
            at.write_tns(t, f)
        out = tmp_path / "factors"
        rc, rep = run(cli, capsys, ["cpd", str(src), "--rank", "3", "--max-iters", "5", "--tol", "0",
                                    "--out-dir", str(out)])
        assert rc == 0 and rep["iterations"] == 5 and len(rep["fit_history"]) == 6
        assert len(rep["factor_files"]) == 3
        f1 = np.loadtxt(rep["factor_files"][0], delimiter=",")
        assert f1.shape == (10, 3)

    def test_check_passes(self, cli, capsys, example_tns):
        rc, rep = run(cli, capsys, ["check", example_tns, "--mode", "2", "--workers", "2"])
        assert rc == 0 and rep["pass"] is True
        assert set(rep["errors"]) == {"seq", "atomic", "buffered"}
