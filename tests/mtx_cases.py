"""Matrix Market test inputs shared by tests/test_mtx.py (CPU: host-side preamble) and
tests/test_gpu_mtx.py (device entry parse).  Every case is judged against the linked reference
read_matrix_market (mmio.cpp:17-55, oracle/_ref) — the expected triplets or error message are
whatever the reference produces on the same bytes."""
import numpy as np

HDR = b"%%MatrixMarket matrix coordinate real general\n"

# Preamble-only cases (no entry line is read): errors and empty matrices.
PREAMBLE_CASES = {
    "empty": b"",
    "bad_banner": b"%%MatrixMarkets matrix coordinate real general\n1 1 0\n",
    "array": b"%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex": b"%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "header_only": HDR,
    "comments_only": HDR + b"% a\n%b\n",
    "blank_lines_then_size": HDR + b"\n\n% c\n\n4 5 0\n",
    "bad_size": HDR + b"4 x 0\n",
    "short_size": HDR + b"4 4\n",
    "zero_nnz": HDR + b"7 3 0\n",
    "zero_nnz_no_newline": HDR + b"7 3 0",
    "crlf_header": b"%%MatrixMarket matrix coordinate real general\r\n2 2 0\r\n",
    "tabs": b"%%MatrixMarket\tmatrix\tcoordinate\tinteger\tgeneral\n\t2\t2\t0\n",
}


def entry_cases():
    """Small files exercising the entry-line grammar (need the device parse)."""
    c = {}
    c["kat"] = HDR + b"% test_storage.cpp:30-36 example\n3 4 4\n1 2 1\n2 1 2\n3 4 3\n1 4 4\n"
    c["symmetric"] = (b"%%MatrixMarket matrix coordinate real symmetric\n4 4 4\n"
                      b"1 1 2.5\n2 1 -1\n4 2 3e-3\n3 3 7\n")
    c["pattern_sym"] = (b"%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n"
                        b"2 1\n3 1 9 junk\n3 3\n")
    c["integer"] = b"%%MatrixMarket matrix coordinate integer general\n2 3 3\n1 1 -7\n2 3 +12\n1 3 0\n"
    c["crlf"] = HDR.replace(b"\n", b"\r\n") + b"2 2 2\r\n1 1 1.5\r\n2 2 -2.25\r\n"
    c["spacing"] = HDR + b"3 3 3\n  1\t 2   0.5  \n\t3 3\t1e2\n 2 2 .5e-1 trailing words\n"
    c["no_final_newline"] = HDR + b"2 2 2\n1 1 1\n2 2 2"
    c["extra_lines_ignored"] = HDR + b"2 2 1\n1 2 4\nthis is not read\n% neither\n"
    c["values_grammar"] = HDR + (
        b"3 3 9\n1 1 1e\n1 2 1e+\n1 3 .\n2 1 -\n2 2 1.5.3\n2 3 0x10\n3 1 1,5\n3 2 inf\n3 3 -0\n")
    c["missing_value"] = HDR + b"2 2 2\n1 1\n2 2 3\n"
    c["extremes"] = HDR + (
        b"3 3 9\n1 1 1e400\n1 2 -1e400\n1 3 1e-400\n2 1 4.9e-324\n2 2 2.4e-324\n"
        b"2 3 2.5e-324\n3 1 1.7976931348623157e308\n3 2 2.2250738585072014e-308\n"
        b"3 3 2.2250738585072011e-308\n")
    c["long_digits"] = HDR + (
        b"2 2 4\n1 1 123456789012345678901234567890\n1 2 0.000000000000000000000000000001234\n"
        b"2 1 3.14159265358979323846264338327950288\n2 2 1.0000000000000000000000000001\n")
    c["int_overflow_row"] = HDR + b"2 2 1\n9223372036854775808 1 1\n"
    c["bad_entry_first"] = HDR + b"3 3 3\n1 1 1\nx 2 2\n9 9 9\n"
    c["out_of_range_first"] = HDR + b"3 3 3\n1 1 1\n4 2 2\nx 2 2\n"
    c["zero_index"] = HDR + b"3 3 1\n0 1 1\n"
    c["float_index"] = HDR + b"3 3 1\n1.0 2 1\n"
    c["blank_entry_line"] = HDR + b"3 3 2\n1 1 1\n\n2 2 2\n"
    c["comment_in_entries"] = HDR + b"3 3 2\n1 1 1\n% late comment\n"
    c["truncated"] = HDR + b"3 3 3\n1 1 1\n2 2 2\n"
    c["truncated_no_newline"] = HDR + b"3 3 3\n1 1 1\n2 2 2"
    c["truncated_after_bad"] = HDR + b"3 3 5\n1 1 1\nbad\n"
    c["size_no_entries"] = HDR + b"3 3 2\n"
    c["size_no_newline"] = HDR + b"3 3 2"
    c["duplicates_kept"] = HDR + b"2 2 3\n1 1 1\n1 1 2\n2 2 3\n"
    return c


def random_real_file(n, m, nnz, seed, fmt="%.17g", symmetric=False):
    """Entries with values spread over many magnitudes, written with printf format `fmt`."""
    rng = np.random.default_rng(seed)
    r = rng.integers(1, n + 1, nnz)
    c = rng.integers(1, m + 1, nnz)
    mant = rng.standard_normal(nnz)
    expo = rng.integers(-320, 300, nnz).astype(np.float64)
    v = mant * np.power(10.0, np.clip(expo, -307, 300)) * np.where(expo < -307, 1e-10, 1.0)
    ints = rng.random(nnz) < 0.2
    v[ints] = np.round(mant[ints] * 100)
    small = rng.random(nnz) < 0.4
    v[small] = rng.standard_normal(int(small.sum()))
    sym = b"symmetric" if symmetric else b"general"
    lines = [b"%%MatrixMarket matrix coordinate real " + sym + b"\n",
             b"%d %d %d\n" % (n, m, nnz)]
    lines += [(b"%d %d " % (a, b)) + (fmt % x).encode() + b"\n" for a, b, x in zip(r, c, v)]
    return b"".join(lines)
