"""CPU: the drop-in dataset ingest (include/hpclust/io.hpp) against the reference's own io.hpp
(compiled here from /root/reference when present): same Dataset values, same error types and
message texts on the same inputs (blank lines, headers, CRLF, other delimiters, ragged rows,
unparseable and non-finite fields, empty files, trailing delimiters)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_INC = Path("/root/reference/proj/include")

PROG = r'''
#include <cstdio>
#include <cstring>
#include "hpclust/io.hpp"
int main(int argc, char** argv) {
    hpclust::TableFormat f;
    f.has_header = argv[2][0] == '1';
    f.delimiter = argv[3][0];
    try {
        hpclust::Dataset d = hpclust::load_dataset(argv[1], f);
        std::printf("ok %zu %zu", d.rows, d.cols);
        for (double v : d.values) std::printf(" %.17g", v);
        std::printf("\n");
        hpclust::save_dataset(d, std::string(argv[1]) + ".out", f);
    } catch (const hpclust::ParseError& e) {
        std::printf("ParseError: %s\n", e.what());
    } catch (const std::exception& e) {
        std::printf("error: %s\n", e.what());
    }
}
'''

CASES = [
    ("plain", "1,2\n3,4\n", "0", ","),
    ("header_crlf_blank", "x,y\r\n1.5,-2e-3\r\n\r\n3,4\r\n", "1", ","),
    ("tabs", "1\t2\t3\n4\t5\t6\n", "0", "\t"),
    ("ragged", "1,2\n3\n", "0", ","),
    ("ragged_bad_extra", "1,2\n3,4,zz\n", "0", ","),
    ("bad_field", "1,2\n3,abc\n", "0", ","),
    ("non_finite", "1,inf\n", "0", ","),
    ("trailing_delim", "1,2,\n", "0", ","),
    ("empty", "", "0", ","),
    ("header_only", "a,b\n", "1", ","),
    ("round_trip", "0.1,1e-300,123456789.123456789\n-0.0,5,6\n", "0", ","),
]


def _build(tmp, name, inc):
    src = tmp / f"{name}.cpp"
    src.write_text(PROG)
    exe = tmp / name
    subprocess.run(["g++", "-O1", "-std=gnu++20", f"-I{inc}", "-o", str(exe), str(src)], check=True,
                   capture_output=True)
    return exe


@pytest.mark.skipif(not REF_INC.exists(), reason="reference headers not present")
def test_io_matches_reference(tmp_path):
    ours = _build(tmp_path, "ours", ROOT / "include")
    ref = _build(tmp_path, "ref", REF_INC)
    for name, text, header, delim in CASES:
        f = tmp_path / f"{name}.csv"
        f.write_bytes(text.encode())
        a = subprocess.run([str(ours), str(f), header, delim], capture_output=True, text=True).stdout
        ao = f.with_suffix(".csv.out").read_bytes() if f.with_suffix(".csv.out").exists() else None
        if ao is not None:
            f.with_suffix(".csv.out").unlink()
        b = subprocess.run([str(ref), str(f), header, delim], capture_output=True, text=True).stdout
        bo = f.with_suffix(".csv.out").read_bytes() if f.with_suffix(".csv.out").exists() else None
        assert a == b, (name, a, b)
        assert ao == bo, name


def test_io_missing_file(tmp_path):
    ours = _build(tmp_path, "ours", ROOT / "include")
    out = subprocess.run([str(ours), str(tmp_path / "nope.csv"), "0", ","], capture_output=True, text=True).stdout
    assert out.strip() == f"ParseError: cannot open file: {tmp_path / 'nope.csv'}"
