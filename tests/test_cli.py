"""CLI: reference-compatible output contract of `primes`,
`verify` and `bench` (reference tests/test_cli.py:29-163) on the GPU engine."""

import json

import numpy as np
import pytest

from paper_2302_10083_b200.cli import main, read_bits


def run(argv, capsys):
    try:
        code = main(argv)
    except SystemExit as exc:
        code = exc.code
    out, err = capsys.readouterr()
    return code, out, err


class TestHost:
    def test_read_bits(self):
        tt = read_bits("0001 0111\n")
        assert tt.n == 3 and tt.support_indices().tolist() == [3, 5, 6, 7]

    def test_bad_input_exit_1(self, capsys, tmp_path):
        p = tmp_path / "x.bits"
        p.write_text("0102")
        assert run(["primes", "--input", str(p)], capsys)[0] == 1
        assert run(["primes"], capsys)[0] == 1  # neither --input nor --n/--density
        assert run(["frobnicate"], capsys)[0] == 1  # usage error


@pytest.mark.gpu
class TestGpu:
    def test_ordering_weight_then_rank(self, capsys, tmp_path):
        p = tmp_path / "t.bits"
        p.write_text("0001100010101011")
        code, out, _ = run(["primes", "--input", str(p)], capsys)
        assert code == 0 and out.splitlines() == ["0**1", "*111", "001*", "1100"]  # tests/test_cli.py:29-35

    def test_majority_and_wildcard_char(self, capsys, tmp_path):
        p = tmp_path / "maj3.bits"
        p.write_text("00010111")
        assert run(["primes", "--input", str(p)], capsys)[1].splitlines() == ["*11", "1*1", "11*"]
        code, out, _ = run(["primes", "--n", "3", "--density", "1", "--wildcard-char", "-"], capsys)
        assert code == 0 and out == "---\n"

    def test_engines_byte_identical(self, capsys):
        base = ["--n", "12", "--density", "0.5", "--seed", "6"]
        outs = {a: run(["primes", "--algo", a, *base], capsys)[1] for a in ("dense", "sparse", "state")}
        assert outs["dense"] == outs["state"] == outs["sparse"] and len(outs["dense"]) > 0

    def test_order_matches_numpy_lexsort(self, pkg, gen_mod):
        from paper_2302_10083_b200.cli import order_for_listing

        r = pkg.dense_prime_ranks(pkg.TruthTable(14, gen_mod.random_words(14, 0.6, 2)))
        w = pkg.rank_weights(r, 14).astype(np.int64)
        assert np.array_equal(order_for_listing(r, 14), r[np.lexsort((r, -w))])

    def test_verify_ok_and_mismatch(self, capsys, monkeypatch):
        code, out, _ = run(["verify", "--n", "11", "--density", "0.6", "--dc", "0.1"], capsys)
        assert code == 0 and out.startswith("OK")
        code, out, _ = run(["verify", "--algo", "dense,sparse,state", "--n", "12", "--density", "0.3"], capsys)
        assert code == 0 and "dense, sparse, state" in out
        monkeypatch.setenv("IMPLICANTS_VERIFY_CORRUPT", "sparse")
        code, _, err = run(["verify", "--n", "11", "--density", "0.6"], capsys)
        assert code == 3 and "MISMATCH" in err

    def test_resource_exit_2(self, capsys):
        code, _, err = run(["primes", "--n", "14", "--density", "0.5", "--mem-cap", "1000"], capsys)
        assert code == 2 and "bytes" in err

    def test_bench_jsonl(self, capsys):
        code, out, _ = run(["bench", "--n", "12..13", "--densities", "0.5,0.9", "--reps", "1"], capsys)
        rows = [json.loads(l) for l in out.splitlines()]
        assert code == 0 and len(rows) == 4
        assert set(rows[0]) == {"engine", "n", "density", "seed", "seconds", "peak_bytes", "prime_count"}

    def test_count_only_matches_readme(self, capsys):
        code, out, _ = run(["primes", "--n", "16", "--density", "0.5", "--seed", "42", "--count-only"], capsys)
        assert code == 0 and out.strip() == "68460"  # pkg/README.md:54-55

    @pytest.mark.parametrize("cfg", [1, 2, 3])
    def test_config_workloads(self, capsys, golden, cfg):
        # BASELINE configs generated on the device (configs.py) -> golden prime counts
        code, out, _ = run(["primes", "--config", str(cfg), "--count-only"], capsys)
        assert code == 0 and int(out) == golden["configs"][str(cfg)]["primes"]


@pytest.mark.gpu
class TestDeviceGenerators:
    """configs.py (product) against oracle/gen.py (checker), byte for byte."""

    @pytest.mark.parametrize("cfg", [1, 2, 3])
    def test_config_values(self, gen_mod, cfg):
        from paper_2302_10083_b200 import configs

        assert np.array_equal(configs.config_values_host(cfg), gen_mod.config_values(cfg))
        assert np.array_equal(configs.config_values_device(cfg).cpu().numpy(), gen_mod.config_values(cfg))

    def test_config4_distribution_small_n(self, gen_mod):
        from paper_2302_10083_b200 import configs

        assert np.array_equal(configs.config_values_host(4, n=14), gen_mod.config_values(4, n=14))

    @pytest.mark.parametrize("seed", [0, 1, 7, 2**63 + 5])
    def test_sbox_seeds(self, gen_mod, seed):
        from paper_2302_10083_b200 import _lib

        out = np.empty(1 << 20, dtype=np.uint8)
        _lib.check(_lib.load().dqmc_gen_sbox_host(out.ctypes.data, seed))
        ref = gen_mod.sbox_complement(seed)
        assert np.array_equal(out, ref) and int((out == 0).sum()) == 1024

    def test_bad_config(self):
        from paper_2302_10083_b200 import configs

        with pytest.raises(ValueError):
            configs.config_values_host(3, n=18)
        with pytest.raises(ValueError):
            configs.config_values_host(9)
