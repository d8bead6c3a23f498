"""End-to-end pipeline on the GPU (cli.run_pipeline), mirroring the
reference's test_cli / acceptance determinism checks: same config -> byte-
identical PNGs; every selector kind renders; usage errors exit 2."""
import numpy as np
import pytest

from paper_1408_0677_b200 import cli

pytestmark = pytest.mark.gpu


def make_cars_like(rows=300, seed=11):
    rng = np.random.default_rng(seed)
    cyl = rng.choice([3, 4, 5, 6, 8], size=rows, p=[0.02, 0.5, 0.02, 0.26, 0.2])
    disp = cyl * 40 + rng.normal(0, 25, rows)
    hp = disp * 0.55 + rng.normal(0, 12, rows)
    weight = 1600 + disp * 4.5 + rng.normal(0, 180, rows)
    accel = 28 - hp * 0.08 + rng.normal(0, 1.6, rows)
    mpg = 48 - weight * 0.008 + rng.normal(0, 2.5, rows)
    year = rng.integers(70, 83, rows)
    origin = rng.choice([1, 2, 3], size=rows, p=[0.62, 0.18, 0.2])
    names = ["mpg", "cylinders", "horsepower", "weight", "acceleration", "year", "origin"]
    return names, np.column_stack([mpg, cyl, hp, weight, accel, year, origin]).astype(float)


@pytest.fixture
def cars_csv(tmp_path):
    names, data = make_cars_like()
    path = tmp_path / "cars.csv"
    with open(path, "w") as fh:
        fh.write(",".join(names) + "\n")
        for row in data:
            fh.write(",".join(f"{v:.6g}" for v in row) + "\n")
    return path


def test_pipeline_deterministic_pngs(cars_csv, tmp_path):
    runs = []
    for tag in ("a", "b"):
        cfg = cli.PipelineConfig(input=str(cars_csv), dims=["mpg", "weight+horsepower", "projection"],
                                 variant="affine", mode="discrete+contour", width=160, height=120,
                                 iterations=60, output=str(tmp_path / f"{tag}-{{dim}}.png"), legend=True)
        paths = cli.run_pipeline(cfg)
        assert len(paths) == 3
        runs.append([open(p, "rb").read() for p in paths])
    assert runs[0] == runs[1]


@pytest.mark.parametrize("variant,mode", [("mean", "contour"), ("linear", "adaptive"), ("rigid", "gradient")])
def test_pipeline_variants(cars_csv, tmp_path, variant, mode):
    cfg = cli.PipelineConfig(input=str(cars_csv), dims=["mpg+weight"], variant=variant, mode=mode,
                             width=96, height=80, iterations=20, output=str(tmp_path / "o-{dim}.png"))
    assert len(cli.run_pipeline(cfg)) == 1


def test_cli_usage_errors_exit_2(cars_csv):
    with pytest.raises(SystemExit) as e:
        cli.main(["--input", str(cars_csv), "--resolution", "bad"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["--input", str(cars_csv), "--dims", "nope"])
    assert e.value.code == 2


def test_cli_missing_file_is_pipeline_error(tmp_path, capsys):
    assert cli.main(["--input", str(tmp_path / "missing.csv")]) == 1
    assert "[dataset]" in capsys.readouterr().err
