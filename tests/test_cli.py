"""CLI parity (reference cli.py): argument handling and exit codes on CPU; verify / count /
multiply / bench driving the engine on the GPU."""
import numpy as np
import pytest

from paper_2309_00628_b200 import cli
from paper_2309_00628_b200.core import Matrix, read_matrix, write_matrix


def test_parse_orders():
    assert cli.parse_orders("2^0..2^4") == [1, 2, 4, 8, 16]
    assert cli.parse_orders("4..32") == [4, 8, 16, 32]
    assert cli.parse_orders("1,2^3,5") == [1, 8, 5]
    for bad in ("3..8", "8..4", "", "0,1"):
        with pytest.raises(ValueError):
            cli.parse_orders(bad)


def test_usage_exit_codes(capsys, tmp_path):
    assert cli.main([]) == cli.EXIT_USAGE
    assert cli.main(["verify", "--orders", "3..5"]) == cli.EXIT_USAGE
    assert cli.main(["count", "--algo", "nope"]) == cli.EXIT_USAGE
    assert "valid presets" in capsys.readouterr().err
    assert cli.main(["verify", "--presets", "strassen,bogus"]) == cli.EXIT_USAGE
    assert cli.main(["count", "--algo", "strassen", "--orders", "6"]) == cli.EXIT_DIMENSION
    assert cli.main(["multiply", str(tmp_path / "missing_a"), str(tmp_path / "missing_b"),
                     "-o", str(tmp_path / "c")]) == cli.EXIT_IO
    (tmp_path / "bad").write_text("1 2\n3\n")
    assert cli.main(["multiply", str(tmp_path / "bad"), str(tmp_path / "bad"), "-o", str(tmp_path / "c")]) == cli.EXIT_IO


def test_svg_renderer():
    svg = cli.render_svg([("a", [(2, 1e-3), (4, 2e-3)]), ("b", [])], "t", "x", "y")
    assert svg.startswith("<svg") and svg.endswith("</svg>") and svg.count("<polyline") == 2


@pytest.mark.gpu
def test_verify_and_count_on_gpu(capsys):
    assert cli.main(["verify", "--orders", "1..64", "--seeds", "1", "--cutoff", "8"]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "0 failures" in out
    assert cli.main(["count", "--algo", "winograd-mod2", "--orders", "2..128"]) == cli.EXIT_OK
    assert "DIVERGED" not in capsys.readouterr().out


@pytest.mark.gpu
def test_multiply_and_bench_on_gpu(tmp_path, capsys):
    rng = np.random.default_rng(7)
    a, b = rng.integers(-8, 9, (37, 50)), rng.integers(-8, 9, (50, 29))
    write_matrix(Matrix(a), str(tmp_path / "a.txt"))
    write_matrix(Matrix(b), str(tmp_path / "b.txt"))
    rc = cli.main(["multiply", str(tmp_path / "a.txt"), str(tmp_path / "b.txt"), "--algo", "winograd-mod2",
                   "--cutoff", "4", "-o", str(tmp_path / "c.txt")])
    assert rc == cli.EXIT_OK
    assert np.array_equal(read_matrix(str(tmp_path / "c.txt")).arr, a @ b)
    rc = cli.main(["multiply", str(tmp_path / "a.txt"), str(tmp_path / "a.txt"), "-o", str(tmp_path / "d.txt")])
    assert rc == cli.EXIT_DIMENSION
    rc = cli.main(["bench", "--presets", "naive,winograd-mod2", "--orders", "2^5..2^7", "--reps", "2",
                   "--csv", str(tmp_path / "b.csv"), "--svg", str(tmp_path / "b.svg")])
    assert rc == cli.EXIT_OK
    lines = (tmp_path / "b.csv").read_text().strip().splitlines()
    assert lines[0].startswith("algo,order") and len(lines) == 1 + 2 * 3
    assert (tmp_path / "b.svg").read_text().count("<polyline") == 2
