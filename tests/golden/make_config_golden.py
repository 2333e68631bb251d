"""Generate tests/golden/config_cases.json from the reference's OWN config parser
(proj/src/config.cpp, compiled in place into oracle/_ref/libref_config.so by oracle/Makefile):
for every config text below, RunConfig::parse_text(text).resolved_text() or the ConfigError
message. tests/test_config.py checks paper_2110_11199_b200.config against it.

Usage (in the build container, where /root/reference is mounted):
    make -C oracle ref && python tests/golden/make_config_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

ACCEPT_TRAIN = ("[run]\nkind = train\nseed = 11\n[engine]\nstrategy = ADPSGD_RM\n"
                "learners = 4\nbatch = 8\nepochs = 2\n[lr]\nbase_lr = 0.05\n"
                "peak_lr = 0.05\n[objective]\nkind = quadratic\ndimension = 6\n"
                "samples = 256\n")  # acceptance.cpp:390-394
ACCEPT_STRAG = ("[run]\nkind = stragglers\nseed = 11\n[engine]\nstrategy = ADPSGD_FM\n"
                "learners = 4\nbatch = 8\nepochs = 1\n[lr]\nbase_lr = 0.02\n"
                "peak_lr = 0.02\n[objective]\nkind = quadratic\ndimension = 6\n"
                "samples = 256\n[cluster]\ncoupled = true\n"
                "[stragglers]\nfactors = 5, 100\n")  # acceptance.cpp:398-404
FULL = """# every key
[run]
kind = stragglers
seed = 9223372036854775807
[engine]
strategy = GENERIC
learners = 5
batch = 32
epochs = 7
staleness_cap = 3
staleness = 0, 1,2 ,3,0
generic_mix = random_ring
[lr]
base_lr = 1e-3
peak_lr = .25
warmup_epochs = 2
anneal_factor = 0.5
anneal_start_epoch = 4
[objective]
kind = mlp
dimension = 12
condition_number = 1e4
noise_sigma = 0
samples = 4096
input_dim = 40
hidden = 256
classes = 32
[cluster]
compute_time = 2.5
comm_pairwise = 0.125
comm_allreduce = 0.3
sync_overhead = 0.01
straggler_learner = 2
straggler_factor = 3.5
coupled = 1
iterations_per_learner = 9
[stragglers]
factors = 2, 5.5,,100 ,
strategies = SDPSGD, ADPSGD_D1D,GENERIC
"""
CASES = {
    "empty": "",
    "acceptance_train": ACCEPT_TRAIN,
    "acceptance_stragglers": ACCEPT_STRAG,
    "full": FULL,
    "crlf_tabs_comments": "[run]\r\n\tkind = train # trailing\r\n  seed=3\r\n# only a comment\r\n\r\n[ engine ]\r\n"
                          "strategy\t=\tADPSGD_D1D\r\nlearners = 8\r\n",
    "last_key_wins": "[engine]\nlearners = 3\nlearners = 6\nstaleness = 1,1\nstaleness = 0\n[stragglers]\nfactors = 3\n",
    "value_with_equals": "[run]\nkind = train\n[objective]\nkind = quadratic\n[engine]\nstrategy = ADPSGD_FM\n"
                         "[cluster]\ncompute_time = 1 = 2\n",
    "signs_and_forms": "[run]\nseed = -1\n[lr]\nbase_lr = +2.\npeak_lr = -0.5e+1\nanneal_factor = 0x1p-1\n"
                       "[cluster]\ncompute_time = inf\ncomm_pairwise = 1E-2\n[engine]\nlearners = +4\nbatch = -2\n",
    "int_wraps": "[engine]\nlearners = 3000000000\nepochs = -4294967295\n",
    "no_trailing_newline": "[engine]\nbatch = 17",
    "straggler_profile": "[engine]\nlearners = 6\n[cluster]\nstraggler_learner = 0\nstraggler_factor = 2\n",
    # errors
    "err_bad_header": "[run\nkind = train\n",
    "err_unknown_section": "[model]\nx = 1\n",
    "err_no_equals": "[run]\nkind train\n",
    "err_unknown_key": "[engine]\nlearner = 4\n",
    "err_unknown_key_no_section": "seed = 4\n",
    "err_bad_double": "[lr]\nbase_lr = fast\n",
    "err_double_trailing": "[lr]\nbase_lr = 0.1x\n",
    "err_double_range": "[lr]\nbase_lr = 1e400\n",
    "err_int_fraction": "[engine]\nbatch = 1.5\n",
    "err_int_exponent": "[engine]\nbatch = 1e3\n",
    "err_int_hex": "[engine]\nbatch = 0x10\n",
    "err_int_empty": "[engine]\nbatch =\n",
    "err_int_range": "[engine]\nbatch = 9223372036854775808\n",
    "err_bool": "[cluster]\ncoupled = yes\n",
    "err_strategy": "[engine]\nstrategy = ADPSGD\n",
    "err_mix": "[engine]\ngeneric_mix = ring\n",
    "err_run_kind": "[run]\nkind = verify\n",
    "err_staleness_item": "[engine]\nstaleness = 1, x\n",
    "err_factor_item": "[stragglers]\nfactors = 5, fast\n",
    "err_strategies_item": "[stragglers]\nstrategies = ADPSGD_FM, SGD\n",
    "err_line_number": "[run]\n\n# c\nkind = train\nseed\n",
}


def main() -> None:
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_config.so"))
    lib.ref_config_resolve.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
    out = {}
    for name, text in CASES.items():
        buf = C.create_string_buffer(1 << 16)
        rc = lib.ref_config_resolve(text.encode(), buf, len(buf))
        out[name] = {"text": text, "rc": rc, "out": buf.value.decode()}
    with open(os.path.join(HERE, "config_cases.json"), "w") as f:
        json.dump({"source": "proj/src/config.cpp via oracle/_ref/libref_config.so", "cases": out}, f, indent=1)
    print(f"{len(out)} cases")


if __name__ == "__main__":
    main()
