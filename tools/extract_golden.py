"""Extract the reference's golden vectors into tests/golden/reference_values.json.

Source: /root/reference/proj/tests/reference_values.hpp (lambda = mu = rho = 1,
omega = 2, "50+ digit arithmetic").  Only the numbers are taken (data, not
code): kHankel (:15-31), kKernels (:35-62), kScalars (:68-110), kIncident
(:114-125), kLogGal (:129-132).  The GPU box has no /root/reference, so the
tests read the committed JSON.
"""
import json
import re
from pathlib import Path

SRC = Path("/root/reference/proj/tests/reference_values.hpp")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "reference_values.json"
NUM = re.compile(r"[-+]?(?:\d+\.\d*|\.\d+|\d+)(?:[eE][-+]?\d+)?")


def block(text, name):
    i = text.index(name)
    j = text.index("{", i)
    depth = 0
    for k in range(j, len(text)):
        if text[k] == "{":
            depth += 1
        elif text[k] == "}":
            depth -= 1
            if depth == 0:
                return text[j:k + 1]
    raise ValueError(name)


def numbers(s):
    s = re.sub(r"//[^\n]*", "", s)
    return [float(x) for x in NUM.findall(s)]


def chunks(v, n):
    assert len(v) % n == 0, (len(v), n)
    return [v[i:i + n] for i in range(0, len(v), n)]


def main():
    t = SRC.read_text()
    hank = [dict(zip(["x", "h0r", "h0i", "h1r", "h1i"], c))
            for c in chunks(numbers(block(t, "kHankel[] =")), 5)]
    kern = []
    for c in chunks(numbers(block(t, "kKernels[] =")), 6 + 24 + 12):
        kern.append(dict(z=c[0:2], m=c[2:4], n=c[4:6], G=c[6:14], D=c[14:22],
                         N=c[22:30], G0=c[30:34], D0=c[34:38], N0=c[38:42]))
    scal = [dict(r=c[0], full=c[1:21], rem=c[21:41], stat=c[41:51])
            for c in chunks(numbers(block(t, "kScalars[] =")), 51)]
    inc = [dict(x=c[0:2], d=c[2:4], n=c[4:6], u=c[6:10], t=c[10:14])
           for c in chunks(numbers(block(t, "kIncident[] =")), 14)]
    loggal = chunks(numbers(block(t, "kLogGal[2][2] =")), 2)
    doc = {"source": "proj/tests/reference_values.hpp", "medium":
           {"lambda": 1.0, "mu": 1.0, "rho": 1.0, "omega": 2.0},
           "hankel": hank, "kernels": kern, "scalars": scal, "incident": inc,
           "log_galerkin": loggal}
    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_text(json.dumps(doc, indent=1))
    print(f"wrote {OUT}: {len(hank)} hankel, {len(kern)} kernels, {len(scal)} scalars, "
          f"{len(inc)} incident")


if __name__ == "__main__":
    main()
