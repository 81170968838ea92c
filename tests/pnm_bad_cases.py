"""Malformed PNM inputs shared by the fixture generator and the tests (the
generator records the reference's error offsets for exactly these)."""

PNM_BAD = [
    b"",                            # missing magic
    b"P3\n2 2\n255\n",              # unsupported magic
    b"P5\n0 2\n255\n",              # width not positive
    b"P5\n2 x\n255\n",              # height not an integer
    b"P5\n2 2\n65535\n",            # maxval
    b"P5\n2 2\n255",                # no whitespace before payload
    b"P5\n2 2\n255\n\x01\x02",      # truncated payload
    b"P6 # c\n2 1 255\n\x01",       # truncated RGB payload after a comment
]
