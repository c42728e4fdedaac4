"""Generates tests/golden/scale.json: per-layer ledgers (all 8 LayerRecord
keys except wall time, batches_sent at workers = 1) and SHA-256 digests of
the full sorted operator at chosen layers, produced by the REFERENCE engine
itself (oracle/_ref/libppref.so, compiled in place from /root/reference by
oracle/build_ref.sh) at the sizes the GPU tests claim:

  chain64_t9            BASELINE config 0 to t = 9 (81,662,152 strings)
  hh_pi4_eps1e-4_t20    BASELINE config-2 member theta_h = pi/4 at eps0 = 1e-4,
                        all 20 steps (<Z62>(20))
  config4_eps1e-4_t8    BASELINE config-4 shape (non-Clifford ZZ, sum Z_i/127)

Digest = sha256(words.tobytes() + coeffs.tobytes()) of the operator exported
sorted ascending by the packed words (word 3 most significant), words as
little-endian uint64[N, 4], coefficients as float64[N] -- the layout
pp_export / Engine.export() return, so the GPU tests hash their own export.

Run here (the reference is single-threaded at workers = 1; chain64_t9 takes
several minutes):   python tests/golden/make_scale_golden.py [case ...]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)
import oracle as O  # noqa: E402
from make_golden import bits, chain_text, hh_text, kicked_gates  # noqa: E402


def digest(words, coeffs):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(words, np.uint64).tobytes())
    h.update(np.ascontiguousarray(coeffs, np.float64).tobytes())
    return h.hexdigest()


CASES = {
    "chain64_t9": dict(text="chain", n=64, thx=0.3, thx_pi=0, thzz=-0.5, thzz_pi=1, init=[(32, 1.0)], eps=0.0,
                       layers=9, digest_at=[4, 7, 8, 9]),
    "hh_pi4_eps1e-4_t20": dict(text="hh", n=127, thx=0.25, thx_pi=1, thzz=-0.5, thzz_pi=1, init=[(62, 1.0)],
                               eps=1e-4, layers=20, digest_at=[6, 8, 12, 16, 20]),
    "config4_eps1e-4_t8": dict(text="hh", n=127, thx=0.4, thx_pi=0, thzz=-np.pi / 2 + 0.2, thzz_pi=0,
                               init=[(q, 1.0 / 127) for q in range(127)], eps=1e-4, layers=8,
                               digest_at=[3, 4, 6, 8]),
}


def run_case(name, spec):
    text = chain_text(64) if spec["text"] == "chain" else hh_text()
    gates = kicked_gates(text, spec["thx"], spec["thx_pi"], spec["thzz"], spec["thzz_pi"])
    r = O.RefEngine(spec["n"], spec["eps"], cadence=0, workers=1, threads=1)
    w = np.stack([O.site_word(s, 3) for s, _ in spec["init"]])
    r.set_initial(w, [c for _, c in spec["init"]])
    rows, digests = [], {}
    t0 = time.time()
    for t in range(1, spec["layers"] + 1):
        row = r.run_circuit(gates, 1)[0]
        rows.append({"t": t, "observable_bits": bits(row["observable"]), "observable": row["observable"],
                     "term_count": row["term_count"], "global_max_bits": bits(row["global_max"]),
                     "removed": row["removed"], "batches_sent": row["batches_sent"],
                     "records_sent": row["records_sent"]})
        if t in spec["digest_at"]:
            ww, cc = r.export()
            digests[str(t)] = digest(ww, cc)
            del ww, cc
        print(f"{name} t={t} |O|={row['term_count']} obs={row['observable']!r} ({time.time() - t0:.0f}s)",
              flush=True)
    out = {k: v for k, v in spec.items() if k != "text"}
    out.update({"geometry": "chain" if spec["text"] == "chain" else "heavy_hex_ref", "rows": rows,
                "digests": digests, "init": [[s, c] for s, c in spec["init"]]})
    return out


def main():
    path = os.path.join(HERE, "scale.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    names = sys.argv[1:] or list(CASES)
    for name in names:
        data[name] = run_case(name, CASES[name])
        with open(path, "w") as f:
            json.dump(data, f, indent=1)


if __name__ == "__main__":
    main()
