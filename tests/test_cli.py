"""Command-line front end (paper_1509_04232_b200/cli.py).

Follows the reference's pkg/tests/test_cli.py: label writers and their
round trip, exit codes for every failure class, argument rules and the
SUPERPIX_WORKERS default run on CPU (no engine is created); segment-mode
outputs (checked against the oracle) and the bench CSV run on a B200.
"""

import os

import numpy as np
import pytest

import oracle  # test infrastructure: the checker
import paper_1509_04232_b200 as spx
from paper_1509_04232_b200.cli import (
    BENCH_HEADER,
    BenchReport,
    BenchRow,
    CliConfig,
    _config_from_args,
    _parse_args,
    main,
    read_labels_csv,
    run_bench,
    write_labels,
)


def _ppm(path, h, w, seed=None, value=None):
    if value is not None:
        data = np.full((h, w, 3), value, dtype=np.uint8)
    else:
        data = np.random.default_rng(seed).integers(0, 256, (h, w, 3), dtype=np.uint8)
    spx.write_ppm(str(path), spx.ImageRGB(data))
    return str(path)


class TestLabelWriters:
    def test_csv_rows(self, tmp_path):
        p = tmp_path / "l.csv"
        write_labels(spx.LabelMap(np.array([[0, 1], [2, 3]], dtype=np.int32)), str(p), "csv")
        assert p.read_text() == "0,1\n2,3\n"

    def test_csv_single_cell(self, tmp_path):
        p = tmp_path / "l.csv"
        write_labels(spx.LabelMap(np.array([[7]], dtype=np.int32)), str(p), "csv")
        assert p.read_text() == "7\n"

    def test_pgm_bytes(self, tmp_path):
        p = tmp_path / "l.pgm"
        write_labels(spx.LabelMap(np.array([[0, 255, 3]], dtype=np.int32)), str(p), "pgm")
        assert p.read_bytes() == b"P5\n3 1\n255\n" + bytes([0, 255, 3])

    def test_pgm_capacity_error_leaves_no_file(self, tmp_path):
        p = tmp_path / "l.pgm"
        with pytest.raises(spx.LabelCapacityError):
            write_labels(spx.LabelMap(np.array([[0, 256]], dtype=np.int32)), str(p), "pgm")
        assert not p.exists()

    def test_unknown_format(self, tmp_path):
        with pytest.raises(ValueError):
            write_labels(spx.LabelMap(np.zeros((2, 2), np.int32)), str(tmp_path / "x"), "png")

    @pytest.mark.parametrize("h,w,seed", [(1, 1, 0), (3, 17, 1), (40, 9, 2)])
    def test_csv_round_trip(self, h, w, seed, tmp_path):
        lab = np.random.default_rng(seed).integers(0, 1 << 30, (h, w)).astype(np.int32)
        p = tmp_path / "r.csv"
        write_labels(spx.LabelMap(lab), str(p), "csv")
        assert np.array_equal(read_labels_csv(str(p)).data, lab)


class TestBenchCsv:
    def test_schema(self):
        rows = (BenchRow("a.ppm", 4, 3, "cuda", 9, 0.5, 0.25, None),
                BenchRow("a.ppm", 4, 3, "cuda-batch", 9, 0.125, 0.0, 4.0))
        assert BenchReport(rows).to_csv() == (
            BENCH_HEADER + "\n" + "a.ppm,4,3,cuda,9,0.500000,0.250000,\n"
            "a.ppm,4,3,cuda-batch,9,0.125000,0.000000,4.000\n")


class TestExitCodes:
    """Failures that are decided before any engine exists (CPU)."""

    def test_missing_input_exits_one_without_outputs(self, tmp_path):
        out = tmp_path / "o"
        assert main(["--input", str(tmp_path / "nope.ppm"), "--out", str(out),
                     "--superpixels", "4"]) == 1
        assert not out.exists() or not os.listdir(out)

    def test_corrupt_ppm_exits_one(self, tmp_path):
        bad = tmp_path / "bad.ppm"
        bad.write_bytes(b"P3\n2 2\n255\n")
        assert main(["--input", str(bad), "--out", str(tmp_path / "o"),
                     "--superpixels", "4"]) == 1

    def test_invalid_settings_exit_two(self, tmp_path):
        inp = _ppm(tmp_path / "i.ppm", 8, 8, value=9)
        assert main(["--input", inp, "--out", str(tmp_path / "o"), "--superpixels", "4",
                     "--compactness", "-1"]) == 2

    def test_requires_out_directory(self, tmp_path):
        inp = _ppm(tmp_path / "i.ppm", 8, 8, value=9)
        assert main(["--input", inp, "--superpixels", "4"]) == 2

    def test_segment_mode_takes_single_superpixel_count(self, tmp_path):
        inp = _ppm(tmp_path / "i.ppm", 8, 8, value=9)
        assert main(["--input", inp, "--out", str(tmp_path / "o"),
                     "--superpixels", "4", "9"]) == 2

    def test_bad_env_value_exits_two(self, tmp_path, monkeypatch):
        monkeypatch.setenv("SUPERPIX_WORKERS", "many")
        inp = _ppm(tmp_path / "i.ppm", 8, 8, value=9)
        assert main(["--input", inp, "--out", str(tmp_path / "o"), "--superpixels", "4"]) == 2

    def test_bad_repeats_and_batch_exit_two(self, tmp_path):
        inp = _ppm(tmp_path / "i.ppm", 8, 8, value=9)
        assert main(["--input", inp, "--superpixels", "4", "--bench", "--repeats", "0"]) == 2
        assert main(["--input", inp, "--superpixels", "4", "--bench", "--batch", "0"]) == 2


class TestArguments:
    def test_size_flags_are_exclusive(self):
        with pytest.raises(SystemExit):
            _parse_args(["--input", "x.ppm", "--superpixels", "4", "--spixel-size", "4"])

    def test_one_size_flag_required(self):
        with pytest.raises(SystemExit):
            _parse_args(["--input", "x.ppm"])

    def test_defaults(self):
        c = _config_from_args(_parse_args(["--input", "x.ppm", "--superpixels", "4"]))
        assert (c.engine, c.formats, c.iters, c.compactness, c.tile_len) == \
            ("cuda", ("csv",), 5, 10.0, 16)
        assert c.connectivity == "weak" and c.color_space == "lab" and not c.perturb

    def test_formats_deduplicated_in_order(self):
        c = _config_from_args(_parse_args(["--input", "x", "--superpixels", "4", "--format",
                                           "pgm", "--format", "csv", "--format", "pgm"]))
        assert c.formats == ("pgm", "csv")

    def test_engine_aliases_accepted(self):
        for e in ("seq", "par", "cuda"):
            assert _config_from_args(_parse_args(
                ["--input", "x", "--superpixels", "4", "--engine", e])).engine == e

    def test_env_default_applies(self, monkeypatch):
        monkeypatch.setenv("SUPERPIX_WORKERS", "3")
        assert _config_from_args(_parse_args(["--input", "x", "--superpixels", "4"])).workers == 3

    def test_flag_beats_env(self, monkeypatch):
        monkeypatch.setenv("SUPERPIX_WORKERS", "3")
        args = _parse_args(["--input", "x", "--superpixels", "4", "--workers", "5"])
        assert _config_from_args(args).workers == 5


@pytest.mark.gpu
class TestSegmentGpu:
    def test_writes_all_formats(self, tmp_path):
        inp = _ppm(tmp_path / "img.ppm", 24, 32, seed=1)
        out = tmp_path / "o"
        assert main(["--input", inp, "--out", str(out), "--superpixels", "12",
                     "--format", "csv", "--format", "overlay"]) == 0
        assert sorted(os.listdir(out)) == ["img_labels.csv", "img_overlay.ppm"]
        ov = spx.load_image(str(out / "img_overlay.ppm"))
        assert (ov.width, ov.height) == (32, 24)

    @pytest.mark.parametrize("extra", [[], ["--connectivity", "strict"],
                                       ["--connectivity", "off", "--color-space", "xyz"],
                                       ["--perturb", "--iters", "3"]])
    def test_csv_matches_oracle(self, tmp_path, extra):
        h, w = 48, 64
        inp = _ppm(tmp_path / "img.ppm", h, w, seed=2)
        out = tmp_path / "o"
        assert main(["--input", inp, "--out", str(out), "--spixel-size", "8", *extra]) == 0
        cfg = _config_from_args(_parse_args(["--input", inp, "--spixel-size", "8", *extra]))
        conn = {"off": 0, "weak": 1, "strict": 2}[cfg.connectivity]
        space = {"rgb": 0, "xyz": 1, "lab": 2}[cfg.color_space]
        rgb = spx.load_image(inp).data
        ol = oracle.segment(rgb, 8, h // 8, w // 8, cfg.compactness, no_iters=cfg.iters,
                            space=space, perturb=cfg.perturb, connectivity=conn)[0]
        assert np.array_equal(read_labels_csv(str(out / "img_labels.csv")).data, ol)

    def test_pgm_capacity_exit_two(self, tmp_path):
        inp = _ppm(tmp_path / "img.ppm", 64, 64, seed=3)
        assert main(["--input", inp, "--out", str(tmp_path / "o"), "--spixel-size", "2",
                     "--format", "pgm"]) == 2

    def test_identical_invocations_are_byte_identical(self, tmp_path):
        inp = _ppm(tmp_path / "img.ppm", 40, 40, seed=4)
        a, b = tmp_path / "a", tmp_path / "b"
        for o in (a, b):
            assert main(["--input", inp, "--out", str(o), "--superpixels", "25",
                         "--format", "csv", "--format", "pgm", "--format", "overlay"]) == 0
        for f in os.listdir(a):
            assert (a / f).read_bytes() == (b / f).read_bytes()

    def test_several_inputs_and_sizes(self, tmp_path):
        ins = [_ppm(tmp_path / f"i{k}.ppm", h, w, seed=k)
               for k, (h, w) in enumerate([(16, 16), (24, 40), (16, 16)])]
        out = tmp_path / "o"
        assert main(["--input", *ins, "--out", str(out), "--spixel-size", "4"]) == 0
        assert sorted(os.listdir(out)) == [f"i{k}_labels.csv" for k in range(3)]


@pytest.mark.gpu
class TestBenchGpu:
    def test_rows_and_speedup(self, tmp_path, capsys):
        inp = _ppm(tmp_path / "img.ppm", 48, 64, seed=9)
        out = tmp_path / "o"
        assert main(["--input", inp, "--superpixels", "12", "48", "--bench", "--repeats", "3",
                     "--batch", "8", "--out", str(out)]) == 0
        text = capsys.readouterr().out
        assert (out / "bench.csv").read_text() == text
        lines = text.strip().splitlines()
        assert lines[0] == BENCH_HEADER and len(lines) == 5
        for k, (one, many) in ((12, lines[1:3]), (48, lines[3:5])):
            a, b = one.split(","), many.split(",")
            assert (a[3], b[3]) == ("cuda", "cuda-batch") and int(a[4]) == int(b[4]) == k
            # (times are printed to 1 us, too coarse to recompute the ratio:
            # test_report_rows checks it on the unrounded values)
            assert a[7] == "" and float(b[7]) > 0

    def test_low_repeats_warns(self, tmp_path, capsys):
        inp = _ppm(tmp_path / "img.ppm", 16, 16, seed=11)
        assert main(["--input", inp, "--superpixels", "4", "--bench", "--repeats", "1",
                     "--batch", "2"]) == 0
        assert "below the recommended minimum" in capsys.readouterr().err

    def test_report_rows(self, tmp_path):
        inp = _ppm(tmp_path / "img.ppm", 16, 16, seed=12)
        cfg = CliConfig(inputs=(inp,), out_dir=None, superpixels=None, spixel_size=4,
                        compactness=10.0, iters=2, color_space="lab", connectivity="weak",
                        min_size=None, perturb=False, engine="cuda", workers=None,
                        tile_len=16, formats=("csv",), bench=True, repeats=3, seed=None,
                        batch=4)
        one, many = run_bench(cfg).rows
        assert one.superpixels == 16 and one.speedup is None
        assert many.speedup == pytest.approx(one.mean_s / many.mean_s, rel=1e-9)
        assert one.mean_s > 0 and many.mean_s > 0


@pytest.mark.gpu
@pytest.mark.parametrize("size,k,iters", [(256, 256, 5), (97, 40, 3)])
def test_kernel_bench_engine_equals_stage_chain(size, k, iters, capsys):
    from paper_1509_04232_b200.kernel_bench import main as kb_main
    assert kb_main(["--size", str(size), "--superpixels", str(k), "--iters", str(iters),
                    "--repeats", "2"]) == 0
    out = capsys.readouterr().out
    assert "labels identical: yes" in out
    for stage in ("convert", "init", "associate", "update", "connectivity", "total"):
        assert stage in out


def test_kernel_bench_synthetic_image_is_the_reference_generator():
    from paper_1509_04232_b200.kernel_bench import synthetic_image
    img = synthetic_image(8, 3)
    want = np.random.default_rng(3).integers(0, 256, size=(8, 8, 3), dtype=np.uint8)
    assert np.array_equal(img.data, want)
