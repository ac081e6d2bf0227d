"""phg_denoise_pgm_file: a binary PGM read in pinned row
chunks overlapped with H2D, denoised on the device, written back while later
chunks come off the device.  The written file must be byte-identical to the
reference's write_pgm(denoise(read_pgm(file)).image) (pgm.hpp:98-150,
denoise.hpp:292-311), stats included; errors keep the reference's texts."""
import re

import numpy as np
import pytest

import paper_1306_5390_b200 as P
from paper_1306_5390_b200._lib import InvalidArgument
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _p5(img, header=None):
    h, w = img.shape
    return (header or f"P5\n{w} {h}\n255\n").encode() + img.tobytes()


@pytest.mark.parametrize("w,h,beta", [(481, 321, 1), (3000, 7000, 1), (1500, 900, 2), (64, 1, 1)])
def test_file_roundtrip_matches_reference(tmp_path, w, h, beta):
    img = O.inject_sp_noise(O.synth_image(w, h, w + h), 0.3, 0.5, 3)
    src, dst = tmp_path / "in.pgm", tmp_path / "out.pgm"
    src.write_bytes(_p5(img, f"P5\n# a comment\n{w}  {h}\n# another\n255\n"))
    stats = P.denoise_pgm_file(str(src), str(dst), P.DenoiseParams(beta=beta))
    ref, ref_stats = O.denoise(img, 20, beta)
    assert dst.read_bytes() == _p5(ref)
    assert [(s.flagged, s.replaced) for s in stats] == ref_stats


def test_reference_error_texts(tmp_path):
    cases = [(b"P6\n1 1\n255\n\x00", "not a PGM stream (expected P2 or P5 magic)"),
             (b"P5\n2 x\n255\n", "malformed PGM header"),
             (b"P5\n2 2\n65535\n\x00", "16-bit PGM unsupported"),
             (b"P5\n2 2\n255\nab", "truncated PGM pixel data"),
             (b"P5\n2 2\n99\nabcd", "PGM pixel value exceeds maxval"),
             (b"P5\n2 2\n255x\x00\x00\x00\x00", "malformed PGM header")]
    for i, (data, msg) in enumerate(cases):
        f = tmp_path / f"bad{i}.pgm"
        f.write_bytes(data)
        with pytest.raises(InvalidArgument, match=re.escape(msg)):
            P.denoise_pgm_file(str(f), str(tmp_path / "o.pgm"))
    with pytest.raises(InvalidArgument, match="cannot open"):
        P.denoise_pgm_file(str(tmp_path / "missing.pgm"), str(tmp_path / "o.pgm"))
