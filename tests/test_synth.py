"""Synthetic-input generators used by the benchmark (CPU only)."""
import numpy as np

from paper_2105_01196_b200 import synth


def test_random_population_shape_and_distinct_columns():
    pop = synth.random_population(5000, 37, 3, 5, seed=1)
    lens = pop.lengths()
    assert len(pop) == 5000 and lens.min() >= 3 and lens.max() <= 5
    assert pop.cols.max() < 37
    for i in range(0, 5000, 7):
        s = pop.sequence(i)
        assert len(set(s.tolist())) == s.size


def test_exact_len_population():
    pop = synth.exact_len_population(300, 64, 50, seed=2)
    assert (pop.lengths() == 50).all()
    for i in range(300):
        assert len(set(pop.sequence(i).tolist())) == 50


def test_planted_matrix_contains_its_trends():
    m, truth = synth.planted_trend_matrix(400, 30, 2, 40, 6, seed=3)
    assert m.dtype == np.float32 and m.shape == (400, 30)
    for rows, cols in truth:
        sub = m[np.ix_(rows, cols)]
        # each member row is a permutation of a sorted sequence along one shared order
        order = np.argsort(sub[0])
        assert (np.diff(sub[:, order], axis=1) >= 0).all()
