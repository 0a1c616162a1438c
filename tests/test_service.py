"""HTTP service (mirrors the reference's tests/test_service.py for the routed
endpoints).  Validation paths run on CPU; the report-producing requests run the
CUDA path and are marked gpu."""
import warnings

import pytest

warnings.filterwarnings("ignore", message=".*httpx2.*")

from fastapi.testclient import TestClient  # noqa: E402

from paper_1509_09308_b200 import __version__  # noqa: E402
from paper_1509_09308_b200.commands import Report  # noqa: E402
from paper_1509_09308_b200.service import create_app  # noqa: E402


@pytest.fixture(scope="module")
def client():
    return TestClient(create_app())


def test_health(client):
    r = client.get("/health")
    assert r.status_code == 200
    body = r.json()
    assert body["status"] == "ok" and body["version"] == __version__


@pytest.mark.parametrize("path,body,code", [
    ("/v1/accuracy", {"suite": "mnist-mlp"}, 400),
    ("/v1/accuracy", {"algos": ["f16x16"], "scale": 0.05}, 400),
    ("/v1/accuracy", {"precision": "fp8", "scale": 0.05}, 422),
    ("/v1/accuracy", {"scale": 0.0}, 422),
    ("/v1/bench", {"algo": "sorcery", "scale": 0.02}, 400),
    ("/v1/bench", {"algo": "f4x4:fp8", "scale": 0.02}, 400),
    ("/v1/bench", {"repeats": 0, "scale": 0.02}, 422),
    ("/v1/bench", {"batch": 0}, 422),
    ("/v1/bench", {"suite": "resnet"}, 400),
])
def test_validation_errors(client, path, body, code):
    r = client.post(path, json=body)
    assert r.status_code == code, r.text


def test_unrouted_endpoints_404(client):
    assert client.get("/v1/complexity/winograd").status_code == 404


def test_report_csv_round_trip():
    rep = Report(columns=("layer", "algo", "msec"), seed=3)
    rep.add("conv1.1", "f2x2", 0.1 + 0.2)
    rep.add("TOTAL", "f2x2", None)
    back = Report.from_csv(rep.to_csv())
    assert back.columns == rep.columns and back.seed == 3 and back.rows == rep.rows


@pytest.mark.gpu
def test_accuracy_endpoint(client):
    r = client.post("/v1/accuracy", json={"scale": 0.05, "algos": ["f2x2", "f4x4:fp16"],
                                          "seed": 3})
    assert r.status_code == 200, r.text
    body = r.json()
    assert body["seed"] == 3
    assert body["columns"] == ["layer", "algo", "precision", "max_abs_err"]
    assert len(body["rows"]) == 10
    assert all(row[3] > 0 for row in body["rows"])
    rep = Report.from_csv(body["csv"])
    assert [list(x) for x in rep.rows] == body["rows"]


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["direct", "f2x2", "f4x4-fx:bf16"])
def test_bench_endpoint(client, algo):
    r = client.post("/v1/bench", json={"scale": 0.02, "repeats": 1, "algo": algo})
    assert r.status_code == 200, r.text
    rows = r.json()["rows"]
    assert rows[-1][0] == "TOTAL"
    assert all(row[3] > 0 for row in rows)
