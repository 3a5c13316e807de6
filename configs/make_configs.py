"""Write the five BASELINE configurations as sdmortar-schema JSON.

The recipe is SURVEY.md section 0.1: Omega = (0, X) x (0, 1), Stokes above
y = 0.5 and Darcy below, an nxs x (nys + nyd) array of equal blocks listed
Stokes rows first (top row first, left to right) then Darcy rows (top to
bottom). The schema is the reference's (config.py:21-23, 110-533).

Run: python configs/make_configs.py  (rewrites configs/cfg{1..5}.json)
"""

import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))

# cfg -> (X, nxs, nys, nyd, nf, regions, collocation, mortar elems)
_LAYERED = {
    1: (1.0, 2, 1, 1, 10, dict(n=1, sigma2=1.0, eta=[0.25, 0.125], n_term=2),
        {"kind": "tensor", "m": 3}, 2),
    2: (1.0, 4, 2, 2, 16, dict(n=2, sigma2=1.5, eta=[0.2, 0.1], n_term=3),
        {"kind": "sparse", "level": 2}, 2),
    3: (2.0, 8, 2, 2, 32, dict(n=4, sigma2=2.0, eta=[0.25, 0.05], n_term=4),
        {"kind": "sparse", "level": 2}, 2),
    4: (2.0, 16, 4, 4, 32, dict(n=8, sigma2=2.0, eta=[0.2, 0.05], n_term=4),
        {"kind": "sparse", "level": 3}, 4),
}


def _num(v):
    return float(round(v, 12))


def layered_config(cfg_id, tol=1e-11):
    X, nxs, nys, nyd, nf, reg, colloc, nm = _LAYERED[cfg_id]
    dx = X / nxs
    hs = 0.5 / nys
    hd = 0.5 / nyd
    nreg = reg["n"]
    rw = X / nreg
    regions = [{"rect": [_num(r * rw), 0.0, _num((r + 1) * rw), 0.5],
                "sigma2": reg["sigma2"], "eta": list(reg["eta"]),
                "n_term": reg["n_term"]} for r in range(nreg)]
    blocks, bcs = [], {}
    sid = 0
    # Stokes rows, top row first
    for row in range(nys):
        y1 = 1.0 - row * hs
        y0 = y1 - hs
        for col in range(nxs):
            x0, x1 = col * dx, (col + 1) * dx
            blocks.append({"rect": [_num(x0), _num(y0), _num(x1), _num(y1)],
                           "physics": "stokes", "mesh": [nf, nf]})
            sides = {}
            if row == 0:
                sides["top"] = {"kind": "stress"}
            if col == 0:
                c = ((y1 - y0) / 2.0) ** 2
                expr = f"({_num(y1)!r}-y)*(y-{_num(y0)!r})/{_num(c)!r}"
                sides["left"] = {"kind": "velocity", "value": [expr, 0]}
            if col == nxs - 1:
                sides["right"] = {"kind": "stress"}
            if sides:
                bcs[str(sid)] = sides
            sid += 1
    # Darcy rows, top to bottom
    for row in range(nyd):
        y1 = 0.5 - row * hd
        y0 = y1 - hd
        for col in range(nxs):
            x0, x1 = col * dx, (col + 1) * dx
            xc = 0.5 * (x0 + x1)
            region = min(int(xc // rw), nreg - 1)
            blocks.append({"rect": [_num(x0), _num(y0), _num(x1), _num(y1)],
                           "physics": "darcy", "mesh": [nf, nf],
                           "kl_region": region})
            if row == nyd - 1:
                bcs[str(sid)] = {"bottom": {"kind": "pressure"}}
            sid += 1
    return {
        "domain": {"blocks": blocks},
        "kl_regions": regions,
        "mean_log_perm": {"kind": "constant", "value": 0.0},
        "collocation": colloc,
        "mortars": {"dd": nm, "sd": nm, "ss": nm, "degree": 1},
        "bcs": bcs,
        "method": "S3",
        "cg": ({"tol": tol, "max_iter": 200000} if cfg_id == 4 else {"tol": tol}),
        "output": {"dir": f"out/cfg{cfg_id}"},
    }


def basis_stress_config():
    """cfg 5: four 64x64 Darcy blocks, one 6-term KL region per block."""
    rects = [[0.0, 0.0, 0.5, 0.5], [0.5, 0.0, 1.0, 0.5],
             [0.0, 0.5, 0.5, 1.0], [0.5, 0.5, 1.0, 1.0]]
    return {
        "domain": {"blocks": [{"rect": r, "physics": "darcy",
                               "mesh": [64, 64], "kl_region": j}
                              for j, r in enumerate(rects)]},
        "kl_regions": [{"rect": r, "sigma2": 1.0, "eta": [0.3, 0.1],
                        "n_term": 6} for r in rects],
        "mean_log_perm": {"kind": "constant", "value": 0.0},
        "collocation": {"kind": "tensor", "m": 1},
        "mortars": {"dd": 8, "degree": 1},
        "bcs": {"0": {"left": {"kind": "pressure", "value": 1.0}},
                "3": {"right": {"kind": "pressure", "value": 0.0}}},
        "method": "S3",
        "cg": {"tol": 1e-11},
        "output": {"dir": "out/cfg5"},
    }


def all_configs():
    out = {f"cfg{k}": layered_config(k) for k in _LAYERED}
    out["cfg5"] = basis_stress_config()
    return out


if __name__ == "__main__":
    for name, cfg in all_configs().items():
        with open(os.path.join(HERE, name + ".json"), "w") as fh:
            json.dump(cfg, fh, indent=1)
            fh.write("\n")
        print("wrote", name)
