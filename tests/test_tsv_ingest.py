"""Matrix ingest: the multi-threaded TSV reader of the C ABI
(ebic_tsv_read, paper_2105_01196_b200/csrc/ebic_tsv.cpp) against the
reference's own parse_matrix_tsv (io.cpp:78-111, linked from oracle/_ref):
bit-identical values on files written by the reference's writer (%.17g), the
same shapes, and the same error messages for every malformed-input rule.  CPU
only: the reader needs no device."""
import numpy as np
import pytest

import oracle
from paper_2105_01196_b200 import EbicError, read_matrix_tsv

pytestmark = pytest.mark.skipif(not oracle.ref_io_available(), reason="reference io.cpp not built (oracle/_ref)")


@pytest.mark.parametrize("shape", [(1, 1), (3, 7), (257, 33), (1000, 64)])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_values_bit_identical_to_reference(tmp_path, shape, threads):
    rng = np.random.default_rng(shape[0] * 31 + shape[1])
    m = rng.standard_normal(shape) * 10.0 ** rng.integers(-300, 300, size=shape)
    m[rng.random(shape) < 0.05] = 0.0
    m.flat[0] = -0.0
    if m.size > 3:
        m.flat[1] = 5e-324  # subnormal
        m.flat[2] = np.float64(np.float32(0.1))
    f = tmp_path / "m.tsv"
    oracle.ref_write_matrix_tsv(f, m)
    want = oracle.ref_parse_matrix_tsv(f)
    got = read_matrix_tsv(f, threads=threads)
    assert got.shape == want.shape == m.shape
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))  # bit for bit, -0.0 included
    assert np.array_equal(got.view(np.uint64), m.view(np.uint64))     # %.17g round-trips


def _same_outcome(path, threads=4):
    try:
        want = oracle.ref_parse_matrix_tsv(path)
        ref_err = None
    except oracle.RefParseError as e:
        want, ref_err = None, str(e)
    try:
        got = read_matrix_tsv(path, threads=threads)
        err = None
    except EbicError as e:
        got, err = None, str(e).split(": ", 1)[1]  # strip "ebic status N: "
    assert (ref_err is None) == (err is None), (ref_err, err)
    if ref_err is not None:
        assert err == ref_err
    else:
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


CASES = {
    "corner_cell": "\tc0\tc1\nr0\t1\t2\nr1\t3\t4\n",
    "no_corner_cell": "c0\tc1\nr0\t1\t2\nr1\t3\t4\n",
    "crlf": "\tc0\tc1\r\nr0\t1.5\t-2\r\nr1\t3\t4e-3\r\n",
    "no_final_newline": "\tc0\nr0\t1\nr1\t2",
    "trailing_empty_lines": "\tc0\nr0\t1\n\n\n",
    "empty_line_inside": "\tc0\nr0\t1\n\nr2\t3\n",
    "ragged": "\tc0\tc1\nr0\t1\t2\nr1\t3\n",
    "non_numeric": "\tc0\tc1\nr0\t1\tx\n",
    "plus_sign": "\tc0\nr0\t+1\n",
    "space": "\tc0\nr0\t 1\n",
    "inf": "\tc0\nr0\tinf\n",
    "nan": "\tc0\tc1\nr0\t1\tnan\n",
    "overflow": "\tc0\nr0\t1e400\n",
    "header_mismatch": "\tc0\tc1\tc2\tc3\nr0\t1\t2\n",
    "only_header": "\tc0\tc1\n",
    "no_values": "\tc0\nr0\nr1\n",
    "empty_file": "",
    "error_order": "\tc0\tc1\nr0\t1\t2\nr1\tx\t2\nr2\t1\n",
    # ExpressionMatrix::validate's label rules (matrix.cpp:43-49)
    "dup_row_label": "\tc0\tc1\nr0\t1\t2\nr1\t3\t4\nr0\t5\t6\n",
    "dup_col_label": "\tc0\tc0\nr0\t1\t2\nr1\t3\t4\n",
    "dup_col_label_no_corner": "c1\tc1\nr0\t1\t2\n",
    "dup_row_before_col": "\tc0\tc0\nr0\t1\t2\nr0\t3\t4\n",
    "dup_first_repeat_wins": "\tc0\nb\t1\na\t2\na\t3\nb\t4\n",
    "dup_empty_labels": "\tc0\n\t1\n\t2\n",
    "parse_error_before_dup": "\tc0\nr0\t1\nr0\tx\n",
    "corner_equals_label": "c0\tc0\tc1\nr0\t1\t2\n",
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_rules_and_messages_match_reference(tmp_path, name):
    f = tmp_path / f"{name}.tsv"
    f.write_bytes(CASES[name].encode())
    _same_outcome(f)


def test_first_error_is_the_sequential_one(tmp_path):
    """Errors in several thread ranges: the one the reference meets first wins."""
    rows = ["\t" + "\t".join(f"c{j}" for j in range(4))]
    for r in range(400):
        vals = ["1.0"] * 4
        if r in (37, 150, 399):
            vals[2] = "oops" if r != 150 else "inf"
        rows.append(f"r{r}\t" + "\t".join(vals))
    f = tmp_path / "m.tsv"
    f.write_text("\n".join(rows) + "\n")
    for t in (1, 2, 7, 16):
        _same_outcome(f, threads=t)


def test_missing_file(tmp_path):
    with pytest.raises(EbicError) as ei:
        read_matrix_tsv(tmp_path / "nope.tsv")
    assert ei.value.status == 7
