"""cmd_bench over every reference algorithm name on the GPU (commands.py:26,
136-178): the Winograd names, the direct algorithms and the FFT comparison
path all run and report a TOTAL row (scaled-down VGG-E so the suite is quick)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["direct", "direct-fp32", "fft", "f2x2", "f4x4-fx",
                                  "f4x4:bf16"])
def test_cmd_bench_runs_every_algorithm(algo):
    import paper_1509_09308_b200 as wb
    rep = wb.cmd_bench(algo=algo, batch=1, repeats=1, scale=0.125)
    assert rep.columns == ("layer", "algo", "batch", "msec", "effective_gflops")
    labels = [r[0] for r in rep.rows]
    assert labels[-1] == "TOTAL" and len(labels) == 10
    assert all(r[3] is not None and r[3] > 0 for r in rep.rows)
    assert all(r[1] == algo for r in rep.rows)


def test_cli_bench_direct(capsys):
    from paper_1509_09308_b200.__main__ import main
    assert main(["bench", "--algo", "direct-fp32", "--scale", "0.125", "--repeats", "1",
                 "--format", "csv"]) == 0
    out = capsys.readouterr().out
    assert "TOTAL,direct-fp32" in out
