"""Synthetic benchmark scenes (the reference's bundled fixtures, scenes.py:68-190).

The coordinates are generated with the same float expressions as the
reference builders so triangles, lights and therefore every label, G-buffer
and light choice match bit-for-bit (pinned by tests/test_host.py against
tests/golden/scenes.npz).  ``boxes_point_scene`` is the C1 fixture: the
boxes scene with each rect light replaced by a point light of intensity
radiance*area at its centroid.
"""

from __future__ import annotations

import numpy as np

ALBEDO = {"floor": [0.73, 0.73, 0.73], "plate": [0.62, 0.32, 0.26],
          "wall": [0.65, 0.6, 0.55], "ceiling": [0.8, 0.8, 0.8]}
TINTS = ([1.0, 0.9, 0.78], [0.82, 1.0, 0.86], [0.8, 0.88, 1.0], [1.0, 0.8, 0.92])


def quad(a, b, c, d) -> list:
    """Loop-ordered quad as two triangles (a,b,c), (a,c,d)."""
    a, b, c, d = (list(map(float, p)) for p in (a, b, c, d))
    return [[a, b, c], [a, c, d]]


def spaced(n: int, lo: float, hi: float) -> list:
    if n == 1:
        return [(lo + hi) / 2.0]
    step = (hi - lo) / (n - 1)
    return [lo + i * step for i in range(n)]


def down_light(cx, cz, y, size, radiance) -> dict:
    h = size / 2.0
    return {"type": "rect", "corner": [cx - h, y, cz - h], "edge_u": [size, 0.0, 0.0],
            "edge_v": [0.0, 0.0, size], "radiance": list(radiance)}


_BOXES = {
    8: dict(nx=4, nz=2, size=0.40, base=16.0, xs=(-1.8, 1.8), zs=(-1.0, 0.0),
            fin_x=[-1.2, 0.0, 1.2], fin_z=[-0.5, 0.6]),
    32: dict(nx=8, nz=4, size=0.28, base=30.0, xs=(-2.1, 2.1), zs=(-1.3, 0.5),
             fin_x=[-1.8 + 0.6 * k for k in range(7)], fin_z=[-1.0, -0.4, 0.2, 0.85]),
}


def boxes_scene(n_lights: int) -> dict:
    """Closed low box with a cubicle grid of dividers under n_lights (8 or 32)
    alternating bright/dim rect lights at y = 1.35."""
    if n_lights not in _BOXES:
        raise ValueError("boxes scene supports 8 or 32 lights")
    p = _BOXES[n_lights]
    fx, zn, zf, wh = 3.0, 3.0, -2.2, 1.5
    box = {
        "floor": quad((-fx, 0, zf), (fx, 0, zf), (fx, 0, zn), (-fx, 0, zn)),
        "ceiling": quad((-fx, wh, zf), (fx, wh, zf), (fx, wh, zn), (-fx, wh, zn)),
    }
    walls = []
    for a, b, c, d in (((-fx, 0, zf), (fx, 0, zf), (fx, wh, zf), (-fx, wh, zf)),
                       ((-fx, 0, zn), (fx, 0, zn), (fx, wh, zn), (-fx, wh, zn)),
                       ((-fx, 0, zf), (-fx, 0, zn), (-fx, wh, zn), (-fx, wh, zf)),
                       ((fx, 0, zf), (fx, 0, zn), (fx, wh, zn), (fx, wh, zf))):
        walls += quad(a, b, c, d)
    fins = []
    z_end = p["fin_z"][-1]
    for x in p["fin_x"]:      # tall x-dividers: hard cut between light columns
        fins += quad((x, 0, zf), (x, 0, z_end), (x, 1.1, z_end), (x, 1.1, zf))
    for z in p["fin_z"]:      # lower z-dividers: soft spill between rows
        fins += quad((-fx, 0, z), (fx, 0, z), (fx, 0.8, z), (-fx, 0.8, z))
    xs, zs = spaced(p["nx"], *p["xs"]), spaced(p["nz"], *p["zs"])
    lights = []
    for i, (zc, xc) in enumerate((z, x) for z in zs for x in xs):
        level = 3.0 if ((i % p["nx"]) + (i // p["nx"])) % 2 == 0 else 0.35
        tint = TINTS[i % len(TINTS)]
        lights.append(down_light(xc, zc, 1.35, p["size"], [p["base"] * level * t for t in tint]))
    return {
        "camera": {"position": [0.0, 1.25, 2.55], "look_at": [0.0, 0.0, -0.9], "up": [0.0, 1.0, 0.0],
                   "fov_deg": 48.0, "width": 320, "height": 180},
        "materials": [{"albedo": ALBEDO[k]} for k in ("floor", "plate", "wall", "ceiling")],
        "meshes": [{"material": 0, "triangles": box["floor"]}, {"material": 1, "triangles": fins},
                   {"material": 2, "triangles": walls}, {"material": 3, "triangles": box["ceiling"]}],
        "lights": lights,
    }


def rooms_scene(n_lights: int = 1024) -> dict:
    """Three rooms split by doorway walls under a 32 x n/32 grid of small lights."""
    nx, nz = 32, max(1, n_lights // 32)
    if nx * nz != n_lights:
        raise ValueError("n_lights must be a multiple of 32")
    x0, x1, z0, z1, h = -4.8, 4.8, -1.7, 1.7, 3.0
    walls = []
    for a, b, c, d in (((x0, 0, z0), (x1, 0, z0), (x1, h, z0), (x0, h, z0)),
                       ((x0, 0, z1), (x1, 0, z1), (x1, h, z1), (x0, h, z1)),
                       ((x0, 0, z0), (x0, 0, z1), (x0, h, z1), (x0, h, z0)),
                       ((x1, 0, z0), (x1, 0, z1), (x1, h, z1), (x1, h, z0))):
        walls += quad(a, b, c, d)
    for xw in (-1.6, 1.6):    # interior dividers with a doorway
        dz0, dz1, dh = -0.4, 0.6, 1.9
        walls += quad((xw, 0, z0), (xw, 0, dz0), (xw, h, dz0), (xw, h, z0))
        walls += quad((xw, 0, dz1), (xw, 0, z1), (xw, h, z1), (xw, h, dz1))
        walls += quad((xw, dh, dz0), (xw, dh, dz1), (xw, h, dz1), (xw, h, dz0))
    room_tint = ([1.0, 0.85, 0.7], [0.95, 0.95, 0.9], [0.7, 0.85, 1.0])
    lights = []
    for zc in spaced(nz, -1.3, 1.3):
        for xc in spaced(nx, -4.5, 4.5):
            room = 0 if xc < -1.6 else (1 if xc < 1.6 else 2)
            lights.append(down_light(xc, zc, 2.8, 0.08, [8.0 * t for t in room_tint[room]]))
    return {
        "camera": {"position": [0.5, 1.6, 1.1], "look_at": [-1.7, 0.3, -0.4], "up": [0.0, 1.0, 0.0],
                   "fov_deg": 60.0, "width": 320, "height": 180},
        "materials": [{"albedo": ALBEDO[k]} for k in ("floor", "plate", "ceiling", "wall")],
        "meshes": [{"material": 0, "triangles": quad((x0, 0, z0), (x1, 0, z0), (x1, 0, z1), (x0, 0, z1))},
                   {"material": 2, "triangles": quad((x0, h, z0), (x1, h, z0), (x1, h, z1), (x0, h, z1))},
                   {"material": 3, "triangles": walls}],
        "lights": lights,
    }


def boxes_point_scene(n_lights: int = 8, width: int = 64, height: int = 64) -> dict:
    """C1 fixture: point lights (intensity = radiance * area) at the rect centroids."""
    d = boxes_scene(n_lights)
    pts = []
    for lt in d["lights"]:
        c, u, v = (np.array(lt[k], float) for k in ("corner", "edge_u", "edge_v"))
        area = float(np.linalg.norm(np.cross(u, v)))
        pts.append({"type": "point", "position": list(c + 0.5 * u + 0.5 * v),
                    "intensity": [area * r for r in lt["radiance"]]})
    d["lights"] = pts
    d["camera"] = dict(d["camera"], width=width, height=height)
    return d


BUILDERS = {
    "boxes8": lambda: boxes_scene(8),
    "boxes32": lambda: boxes_scene(32),
    "rooms128": lambda: rooms_scene(128),
    "rooms1k": lambda: rooms_scene(1024),
    "pboxes8": lambda: boxes_point_scene(8),
}
