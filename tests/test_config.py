"""Config front-end and CLI (CPU): paper_2110_11199_b200.config against the reference's own parser
(proj/src/config.cpp, compiled in place -> tests/golden/config_cases.json), the blstm extension,
and the CLI's usage / config-error exit codes (tools/main.cpp:26-29, 266-283)."""
import json
import os

import pytest

from paper_2110_11199_b200 import Precision, Strategy
from paper_2110_11199_b200.cli import EXIT_USAGE, main
from paper_2110_11199_b200.config import RunConfig, split_train_count
from paper_2110_11199_b200.errors import ConfigError

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "config_cases.json")))["cases"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_parser_matches_reference_config_cpp(name):
    c = CASES[name]
    if c["rc"] == 0:
        assert RunConfig.parse_text(c["text"]).resolved_text() == c["out"]
    else:
        assert c["rc"] == 1
        with pytest.raises(ConfigError) as e:
            RunConfig.parse_text(c["text"])
        assert str(e.value) == c["out"]


def test_resolved_text_round_trips():
    # (a seed >= 2^63 resolves to a number std::stol -- and so the reference itself -- cannot read back)
    for c in CASES.values():
        if c["rc"] == 0 and "seed = 1844674407370955" not in c["out"]:
            once = RunConfig.parse_text(c["text"]).resolved_text()
            assert RunConfig.parse_text(once).resolved_text() == once


def test_derived_fields():
    c = RunConfig.parse_text(CASES["straggler_profile"]["text"])
    assert c.cluster.learners == 6 and c.cluster.stragglers == [(0, 2.0)]
    c = RunConfig.parse_text(CASES["full"]["text"])
    assert c.strategy.seed == c.seed == (1 << 63) - 1
    assert c.strategy.strategy == Strategy.GENERIC and c.strategy.staleness == [0, 1, 2, 3, 0]
    assert c.straggler_factors == [2.0, 5.5, 100.0] and c.coupled


def test_blstm_objective_extension():
    text = ("[run]\nseed = 5\n[engine]\nstrategy = ADPSGD_FM\nlearners = 3\nbatch = 4\n[objective]\nkind = blstm\n"
            "layers = 2\nhidden = 32\nbidirectional = true\ninput_dim = 20\nproj = 16\nclasses = 24\nunroll = 6\n"
            "samples = 40\nprecision = fp32\n")
    c = RunConfig.parse_text(text)
    m = c.objective.model()
    assert (m.layers, m.hidden, m.bidirectional, m.input_dim, m.proj, m.classes, m.unroll) == (2, 32, True, 20, 16, 24, 6)
    assert c.objective.precision_enum() == Precision.FP32
    assert c.objective.train_count() == 36  # objectives.cpp:18-23: lround(40 * 0.1) = 4 held out
    again = RunConfig.parse_text(c.resolved_text())
    assert again.resolved_text() == c.resolved_text() and again.objective.model() == m
    with pytest.raises(ConfigError, match="toy objectives"):
        RunConfig.parse_text("[objective]\nkind = mlp\n").objective.model()
    with pytest.raises(ConfigError, match="quadratic, logistic, mlp or blstm"):
        RunConfig.parse_text("[objective]\nkind = lstm\n")
    with pytest.raises(ConfigError, match="fp32 or bf16"):
        RunConfig.parse_text("[objective]\nprecision = tf32\n")


def test_split_train_count():
    assert split_train_count(256) == 230  # lround(25.6) = 26
    assert split_train_count(25) == 22    # lround(2.5) = 3 (half away from zero)
    assert split_train_count(3) == 2 and split_train_count(2) == 1


def test_cli_usage_and_config_errors(tmp_path, capsys):
    assert main([]) == EXIT_USAGE
    assert main(["train"]) == EXIT_USAGE  # --config is required
    assert main(["verify"]) == EXIT_USAGE
    assert main(["train", "--config", str(tmp_path / "missing.ini")]) == EXIT_USAGE
    assert "cannot open config file" in capsys.readouterr().err
    bad = tmp_path / "bad.ini"
    bad.write_text("[engine]\nstrategy = ADPSGD_FM\nlearners = 2\n[objective]\nkind = blstm\n")
    assert main(["train", "--config", str(bad), "--out", str(tmp_path / "o")]) == EXIT_USAGE
    assert "FM/RM mixing requires at least 3 learners" in capsys.readouterr().err
