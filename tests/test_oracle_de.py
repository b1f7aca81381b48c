"""CPU: the C restatement of the DE generation (oracle/evb_oracle.c) pinned bit-for-bit against the
reference engine itself (oracle/_ref: de_builder-built de_engine<double> stepped with
rng_stream::scripted), and KATs from tests/test_de.cpp."""
import numpy as np
import pytest

import oracle as O
from paper_2505_17430_b200.de import DEConfig, preset_de, preset_jade, preset_shade

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def run_both(cfg, P, D, kind, gens, seed, lb=-100.0, ub=100.0, scale=1.0):
    o, m = O.shift_rotation(seed, D)
    m = m * scale
    ref = O.RefDE(cfg, P, D)
    ref.set_problem_base(kind, o, m, 0.0)
    orc = O.OracleDE(cfg, P, D)
    orc.set_problem_base(kind, o, m, 0.0)
    rng = np.random.default_rng(seed)
    x = rng.uniform(lb, ub, size=(P, D))
    fit = O.eval_batch(kind, o, m, 0.0, x)
    ref.set_pop(x, fit)
    orc.set_state(x, fit)
    for g in range(gens):
        words = rng.integers(0, 2**64 - 1, size=P * (2 * D + 40) + 64, dtype=np.uint64, endpoint=True)
        out = orc.generation(words, lb, ub)
        n_used = int(out["words"].sum() + out["archive_words"])
        assert ref.generation(words[:n_used], lb, ub), f"gen {g}: reference consumed a different word count"
        st = ref.get()
        assert np.array_equal(st["pop"], orc.pop), g
        assert np.array_equal(st["fit"], orc.fit), g
        assert st["archive_size"] == orc.s.arch_size
        assert np.array_equal(st["archive"], orc.archive[:orc.s.arch_size])
        if cfg.parameter != "fixed":
            assert np.array_equal(st["memory_f"], orc.mem_f) and np.array_equal(st["memory_cr"], orc.mem_cr)
            assert st["write_index"] == orc.s.write_index


@pytest.mark.parametrize("cfg,kind,scale", [
    (preset_de(0.5, 0.9), 5, 0.0512),          # config 0 construction
    (preset_shade(0.11, 40, 1.0), 6, 1.0),      # config 2 construction (smaller)
    (preset_jade(0.05, 0.1, 0.5), 0, 1.0),
    (DEConfig("best_1", "binomial", "reflect", "fixed", f=0.7, cr=0.3), 1, 1.0),
    # exponential crossover (de/strategy.hpp:199-216) and reinitialize repair (:279-290)
    (DEConfig("rand_1", "exponential", "clip", "fixed", f=0.5, cr=0.9), 5, 1.0),
    (DEConfig("rand_1", "binomial", "reinitialize", "fixed", f=0.9, cr=0.9), 6, 1.0),
    (DEConfig("ttpb_1", "exponential", "reinitialize", "shade", p_best=0.11, use_archive=True, memory_size=10,
              archive_rate=1.0), 0, 1.0),
])
def test_c_restatement_matches_reference_engine(cfg, kind, scale):
    run_both(cfg, 40, 12, kind, 6, 3, scale=scale)


def test_native_stream_config0():
    # BASELINE config 0: rand/1/bin, F 0.5, CR 0.9, D=10, pop=100, rastrigin on 0.0512 M (x - o),
    # draws from rng_stream(42, 0): init_population, evaluation, one generation
    P, D = 100, 10
    o, m = O.shift_rotation(42, D)
    m = m * 0.0512
    ref = O.RefDE(preset_de(), P, D)
    ref.set_problem_base(5, o, m, 0.0)
    ref.native_run(42, 0, 1, -100.0, 100.0)
    st = ref.get()
    words = O.rng_words(42, 0, P * D + P * (D + 20))
    x0 = np.empty((P, D))
    rng = __import__("ctypes").create_string_buffer(O.C().orc_rng_size())
    O.C().orc_rng_scripted(rng, O.ptr(words), len(words))
    O.C().orc_init_population(rng, P, D, -100.0, 100.0, O.ptr(x0))
    orc = O.OracleDE(preset_de(), P, D)
    orc.set_problem_base(5, o, m, 0.0)
    orc.set_state(x0, O.eval_batch(5, o, m, 0.0, x0))
    out = orc.generation(words[P * D:], -100.0, 100.0)
    assert np.array_equal(st["pop"], orc.pop)
    assert np.array_equal(st["fit"], orc.fit)
    # donor indices distinct from the target and from each other (de/strategy.hpp:84-86)
    idx = out["idx"]
    for i in range(P):
        a, b, c = idx[i, :3]
        assert len({i, a, b, c}) == 4


def test_rand1_kat_via_generation():
    # tests/test_de.cpp:52-71: pop {{1,1},{2,0},{0,0},{5,5}}, target 3, r1=0 r2=1 r3=2, F=0.5
    # -> donor {2, 1}; with CR = 1 the trial is the donor.
    P, D = 4, 2
    cfg = DEConfig("rand_1", "binomial", "clip", "fixed", f=0.5, cr=1.0)
    orc = O.OracleDE(cfg, P, D)
    orc.set_problem_base(0, np.zeros(2), np.eye(2), 0.0)
    x = np.array([[1.0, 1.0], [2.0, 0.0], [0.0, 0.0], [5.0, 5.0]])
    fit = np.array([2.0, 4.0, 0.0, 50.0])
    orc.set_state(x, fit)

    def idx_word(k, n):  # tests/support/forcing.hpp:12-15
        return ((k << 64) + (1 << 63)) // n

    words = []
    for i in range(P):
        r = [v for v in range(P) if v != i][:3]
        words += [idx_word(r[0], P), idx_word(r[1], P), idx_word(r[2], P), idx_word(0, D), 0, 0]
    out = orc.generation(np.array(words, np.uint64), -100.0, 100.0)
    assert list(out["idx"][3, :3]) == [0, 1, 2]
    assert np.array_equal(orc.pop[3], [2.0, 1.0])  # 26 -> 5 improves, trial kept
