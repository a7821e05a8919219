"""Config-driven runner (next-row f4): the reference's INI configs, methods and
deterministic CSV/JSON outputs (config.hpp/.cpp, runner.hpp/.cpp), running on
the B200 path, plus a `biewos_dtn` method for the BASELINE configurations.

  RawConfig, parse_config_text/file, apply_override   config.cpp:100-182
  scene_from_config                                   runner.cpp:303-343
  run(cfg) -> RunRecord (csv_text, json_text)         runner.cpp:345-390
  write_outputs, compare_csv                          runner.cpp:392-479
Methods: biewos_point, last_passage, field_eval, biewos_patch, biewos_dtn,
biewos_pipeline (config 5); `[gpu] devices` runs the last two on a device group
(bw_group_*) with the same results. `wos.workers`
is excluded from the config echo so outputs never depend on it
(config.cpp:122).
"""
from __future__ import annotations

import itertools
import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import ApplicabilityError, ConfigError

VERSION = "biewos-b200 1"


def _trim(s: str) -> str:
    return s.strip(" \t\r\n")


def _split_tokens(s: str) -> list:
    """Whitespace- or comma-separated tokens; ';' is a token of its own."""
    out, cur = [], ""
    for ch in s:
        if ch in " \t,":
            if cur:
                out.append(cur)
                cur = ""
        elif ch == ";":
            if cur:
                out.append(cur)
                cur = ""
            out.append(";")
        else:
            cur += ch
    if cur:
        out.append(cur)
    return out


@dataclass
class RawConfig:  # config.hpp:13-40
    data: dict = field(default_factory=dict)
    line_of: dict = field(default_factory=dict)
    name: str = "<config>"

    def has(self, sec, key) -> bool:
        return key in self.data.get(sec, {})

    def fail(self, sec, key, what):
        line = self.line_of.get(sec, {}).get(key, 0)
        where = f"{self.name}:{line}: " if line else f"{self.name}: "
        raise ConfigError(f"{where}[{sec}] {key}: {what}")

    def tokens(self, sec, key):
        if not self.has(sec, key):
            raise ConfigError(f"{self.name}: missing [{sec}] {key}")
        return self.data[sec][key]

    def get_str(self, sec, key, dflt=None):
        if dflt is not None and not self.has(sec, key):
            return dflt
        t = self.tokens(sec, key)
        if len(t) != 1:
            self.fail(sec, key, "expected a single value")
        return t[0]

    def get_real(self, sec, key, dflt=None):
        if dflt is not None and not self.has(sec, key):
            return float(dflt)
        s = self.get_str(sec, key)
        try:
            return float(s)
        except ValueError:
            self.fail(sec, key, f"not a number: '{s}'")

    def get_int(self, sec, key, dflt):
        if not self.has(sec, key):
            return int(dflt)
        v = self.get_real(sec, key)
        if v != int(v):
            self.fail(sec, key, "expected an integer")
        return int(v)

    def get_bool(self, sec, key, dflt):
        if not self.has(sec, key):
            return bool(dflt)
        s = self.get_str(sec, key).lower()
        if s in ("1", "true", "yes", "on"):
            return True
        if s in ("0", "false", "no", "off"):
            return False
        self.fail(sec, key, f"not a boolean: '{s}'")

    def get_list(self, sec, key, dflt=None):
        if dflt is not None and not self.has(sec, key):
            return list(dflt)
        out = []
        for s in self.tokens(sec, key):
            try:
                out.append(float(s))
            except ValueError:
                self.fail(sec, key, f"not a number: '{s}'")
        return out

    def echo(self) -> str:  # config.cpp:117-129
        parts = []
        for sec in sorted(self.data):
            for key in sorted(self.data[sec]):
                if (sec == "wos" and key == "workers") or sec == "gpu":
                    continue  # speed only, never results (device lists included)
                parts.append(f"{sec}.{key}=" + " ".join(self.data[sec][key]))
        return ";".join(parts)


def parse_config_text(text: str, name: str = "<config>") -> RawConfig:  # config.cpp:131-163
    cfg = RawConfig(name=name)
    section = ""
    for lineno, line in enumerate(text.splitlines(), 1):
        if "#" in line:
            line = line[: line.index("#")]
        line = _trim(line)
        if not line:
            continue
        if line[0] == "[":
            if line[-1] != "]":
                raise ConfigError(f"{name}:{lineno}: malformed section header")
            section = _trim(line[1:-1])
            if not section:
                raise ConfigError(f"{name}:{lineno}: empty section name")
            cfg.data.setdefault(section, {})
            continue
        if "=" not in line:
            raise ConfigError(f"{name}:{lineno}: expected 'key = value'")
        if not section:
            raise ConfigError(f"{name}:{lineno}: key outside any section")
        key = _trim(line[: line.index("=")])
        if not key:
            raise ConfigError(f"{name}:{lineno}: empty key")
        cfg.data[section][key] = _split_tokens(_trim(line[line.index("=") + 1:]))
        cfg.line_of.setdefault(section, {})[key] = lineno
    return cfg


def parse_config_file(path: str) -> RawConfig:
    try:
        with open(path) as f:
            return parse_config_text(f.read(), path)
    except OSError:
        raise ConfigError(f"cannot open config file: {path}")


def apply_override(cfg: RawConfig, spec: str) -> None:  # config.cpp:173-182
    eq, dot = spec.find("="), spec.find(".")
    if eq < 0 or dot < 0 or dot > eq:
        raise ConfigError(f"--set expects section.key=value, got '{spec}'")
    sec, key = spec[:dot], spec[dot + 1: eq]
    cfg.data.setdefault(sec, {})[key] = _split_tokens(spec[eq + 1:])
    cfg.line_of.setdefault(sec, {})[key] = 0


# ---------------------------------------------------------------------------
@dataclass
class RunRecord:  # runner.hpp:13-30
    method: str = ""
    schema: str = ""
    columns: list = field(default_factory=list)
    rows: list = field(default_factory=list)
    paths_total: float = 0.0
    wall_seconds: float = 0.0
    row_seconds: list = field(default_factory=list)
    csv_text: str = ""
    json_text: str = ""


def _vec(v, what):
    if len(v) == 2:
        return (v[0], v[1], 0.0)
    if len(v) == 3:
        return tuple(v)
    raise ConfigError(f"{what}: expected 2 or 3 coordinates")


def _wos(cfg: RawConfig, seed=None, workers=None):
    from .wos import WosConfig

    w = WosConfig(eps_shell=cfg.get_real("wos", "eps_shell", 1e-5),
                  trunc_radius=cfg.get_real("wos", "trunc_radius", 1e5),
                  max_steps=cfg.get_int("wos", "max_steps", 10000),
                  seed=cfg.get_int("wos", "seed", 0), workers=cfg.get_int("wos", "workers", 1))
    if seed is not None:
        w.seed = seed
    if workers is not None:
        w.workers = workers
    return w


def scene_from_config(cfg: RawConfig):  # runner.cpp:303-343
    from .geometry import DomainSide, PointSource, Scene, SinSin

    kind = cfg.get_str("scene", "kind")
    if kind == "half_space":
        h = cfg.get_real("scene", "charge_height", 1.0)
        scale = cfg.get_real("scene", "charge_scale", 1.0)
        plane = cfg.get_real("scene", "plane_z", 0.0)
        return Scene.half_space(plane, PointSource(q=scale, s=(0.0, 0.0, plane - h)))
    if kind == "four_plates":
        v = cfg.get_list("scene", "potentials", [1, 0, 0, 0])
        if len(v) != 4:
            cfg.fail("scene", "potentials", "expected four values")
        return Scene.four_plates(v)
    if kind == "thin_disk":
        return Scene.thin_disk(cfg.get_real("scene", "b", 1.0), cfg.get_real("scene", "potential", 1.0))
    if kind == "sphere":
        R = cfg.get_real("scene", "R", 1.0)
        side = DomainSide.Interior if cfg.get_str("scene", "side", "exterior") == "interior" \
            else DomainSide.Exterior
        if cfg.has("scene", "charge"):
            return Scene.sphere(R, side, cfg.get_real("scene", "charge") / (4.0 * math.pi * R))
        return Scene.sphere(R, side, cfg.get_real("scene", "potential", 1.0))
    if kind == "four_plates_sine":  # runner.cpp:318-324
        m, n = cfg.get_real("scene", "m", 1.0), cfg.get_real("scene", "n", 1.0)
        plates = [[0, 1, 0, 1], [-1, 0, 0, 1], [-1, 0, -1, 0], [0, 1, -1, 0]]
        return Scene.plate_set(plates, SinSin(1.0, (m, n)))
    cfg.fail("scene", "kind", f"unknown scene kind '{kind}'")


def _analytic_point(cfg, scene, x):  # runner.cpp:55-72
    from .geometry import SceneKind

    if scene.kind == SceneKind.HalfSpace:
        h = cfg.get_real("scene", "charge_height", 1.0)
        scale = cfg.get_real("scene", "charge_scale", 1.0)
        return scale * h / (x[0] ** 2 + x[1] ** 2 + h * h) ** 1.5
    if scene.kind == SceneKind.ThinDisk:
        b, v = scene.disk_radius, scene.feature_potential[0]
        rho = math.hypot(x[0], x[1])
        if rho >= b:
            return None
        return 8.0 * b * v / (4.0 * math.pi * b * math.sqrt(b * b - rho * rho))
    return None


def _reference(cfg, scene, x):  # runner.cpp:74-88
    mode = cfg.get_str("method", "reference", "none")
    if mode == "none":
        return None
    if mode == "analytic":
        r = _analytic_point(cfg, scene, x)
        if r is None:
            cfg.fail("method", "reference", "no analytic reference for this scene")
        return r
    try:
        return float(mode)
    except ValueError:
        cfg.fail("method", "reference", "expected 'analytic', 'none' or a number")


def _err_pct(v, ref):
    return float("nan") if not ref else (v / ref - 1.0) * 100.0


def _nan(ref):
    return float("nan") if ref is None else ref


def _run_point(cfg, scene, rec, seed, workers):  # runner.cpp:115-149
    from .point_solver import HemisphereFrame, solve_point

    x = _vec(cfg.get_list("method", "x"), "method.x")
    axis = np.asarray(_vec(cfg.get_list("method", "axis", [0, 0, 1]), "method.axis"), float)
    axis = axis / np.linalg.norm(axis)
    base = _wos(cfg, seed, workers)
    ref = _reference(cfg, scene, x)
    rec.schema = "biewos_point/v1"
    rec.columns = ["a", "delta_frac", "n_g1", "n_g2", "n_path", "seed", "sigma1", "sigma2",
                   "total", "se", "ref", "err_pct", "paths"]
    sweeps = itertools.product(cfg.get_list("method", "a"),
                               cfg.get_list("method", "delta_frac", [1e-4]),
                               cfg.get_list("method", "n_g1", [20]),
                               cfg.get_list("method", "n_g2", [20]),
                               cfg.get_list("method", "n_path", [1000]))
    for row, (a, df, g1, g2, npath) in enumerate(sweeps):
        t0 = time.perf_counter()
        w = _wos(cfg, seed, workers)
        w.n_paths, w.seed = int(npath), base.seed + row
        r = solve_point(scene, HemisphereFrame(x, a, tuple(axis)), int(g1), int(g2), df * a, w)
        paths = g1 * g1 * npath
        rec.rows.append([a, df, g1, g2, npath, w.seed, r.sigma1, r.sigma2, r.total, r.std_error,
                         _nan(ref), _err_pct(r.total, ref), paths])
        rec.paths_total += paths
        rec.row_seconds.append(time.perf_counter() - t0)


def _run_lp(cfg, scene, rec, seed, workers):  # runner.cpp:151-179
    from .last_passage import estimate_lp
    from .point_solver import HemisphereFrame

    x = _vec(cfg.get_list("method", "x"), "method.x")
    axis = np.asarray(_vec(cfg.get_list("method", "axis", [0, 0, 1]), "method.axis"), float)
    axis = axis / np.linalg.norm(axis)
    allow = cfg.get_bool("method", "allow_general_data", False)
    base = _wos(cfg, seed, workers)
    ref = _reference(cfg, scene, x)
    rec.schema = "last_passage/v1"
    rec.columns = ["a", "n_path", "seed", "sigma_lp", "se", "n_inf", "ref", "err_pct", "paths"]
    sweeps = itertools.product(cfg.get_list("method", "a"),
                               cfg.get_list("method", "n_path", [400000]))
    for row, (a, npath) in enumerate(sweeps):
        t0 = time.perf_counter()
        w = _wos(cfg, seed, workers)
        w.seed = base.seed + row
        r = estimate_lp(scene, HemisphereFrame(x, a, tuple(axis)), int(npath), w, allow)
        rec.rows.append([a, npath, w.seed, r.sigma_lp, r.std_error, r.n_infinity, _nan(ref),
                         _err_pct(r.sigma_lp, ref), npath])
        rec.paths_total += npath
        rec.row_seconds.append(time.perf_counter() - t0)


def _run_field_eval(cfg, scene, rec):  # runner.cpp:243-299
    from .field_eval import evaluate_batch
    from .geometry import DomainSide, SceneKind

    if scene.kind != SceneKind.Sphere or not scene.piecewise_const:
        raise ConfigError("field_eval demo expects a constant-potential sphere scene")
    R, V = scene.sphere_radius, scene.feature_potential[0]
    toks, targets, cur = cfg.tokens("method", "targets"), [], []
    for t in toks:
        if t == ";":
            if cur:
                targets.append(_vec(cur, "method.targets"))
            cur = []
            continue
        cur.append(float(t))
        if len(cur) == 3:
            targets.append(tuple(cur))
            cur = []
    if cur:
        targets.append(_vec(cur, "method.targets"))
    rec.schema = "field_eval/v1"
    rec.columns = ["n_panels", "tx", "ty", "tz", "u", "ref", "err_pct"]
    for nf in cfg.get_list("method", "n_panels", [2000]):
        t0 = time.perf_counter()
        nlat = max(4, int(math.sqrt(nf / 2.0)))
        nlon = 2 * nlat
        P = []
        for i in range(nlat):
            th0, th1 = math.pi * i / nlat, math.pi * (i + 1) / nlat
            thc = 0.5 * (th0 + th1)
            band = (math.cos(th0) - math.cos(th1)) * 2.0 * math.pi / nlon * R * R
            for j in range(nlon):
                ph = 2.0 * math.pi * (j + 0.5) / nlon
                n = (math.sin(thc) * math.cos(ph), math.sin(thc) * math.sin(ph), math.cos(thc))
                P.append([R * n[0], R * n[1], R * n[2], *n, band, V, -V / R])
        u, _ = evaluate_batch(np.array(P), np.array(targets), flag_near=False)
        for t, ut in zip(targets, u):
            ref = None
            if scene.side == DomainSide.Exterior:
                r = math.sqrt(sum(c * c for c in t))
                ref = V * R / r if r > R else 0.0
            rec.rows.append([len(P), *t, ut, _nan(ref), _err_pct(ut, ref)])
        rec.row_seconds.append(time.perf_counter() - t0)


def _run_patch(cfg, scene, rec, seed):  # runner.cpp:181-225
    """biewos_patch: the Neumann field over one sphere patch (solve_patch through
    bw_solve_patch). The Gamma quadrature is the GL x uniform WOS node rule of
    the DtN path on grid_ntheta x grid_nphi nodes (the reference interpolates a
    uniform grid instead); meshes beyond 64 panels (the
    reference's 16 x 36 default) take the large-patch kernels."""
    from .dtn import BIE_FIRST, BIE_SECOND, DtnConfig, PATCH_DTYPE, solve_patch
    from .geometry import DomainSide, SceneKind
    from .nodes import gamma_rule, wos_patch_nodes

    if scene.kind != SceneKind.Sphere:
        raise ConfigError("biewos_patch expects a sphere scene")
    R = scene.sphere_radius
    center = np.asarray(_vec(cfg.get_list("method", "center", [0, 0, R]), "method.center"), float)
    a = cfg.get_real("method", "a", 1.0)
    bands = cfg.get_int("method", "bands", 16)
    az = cfg.get_int("method", "azimuth", 36)
    nt = cfg.get_int("method", "grid_ntheta", 64)
    nphi = cfg.get_int("method", "grid_nphi", 128)
    kind_s = cfg.get_str("method", "kind", "second")
    if kind_s not in ("first", "second"):
        cfg.fail("method", "kind", f"expected first or second, got '{kind_s}'")
    dcfg = DtnConfig(bands=bands, azimuth=az, kind=BIE_FIRST if kind_s == "first" else BIE_SECOND)
    w = _wos(cfg, seed, None)
    w.n_paths = cfg.get_int("method", "n_path", 10000)
    ref = None
    mode = cfg.get_str("method", "reference", "none")
    if mode == "analytic":
        if not scene.piecewise_const:
            cfg.fail("method", "reference", "analytic patch reference needs constant data")
        ref = -scene.feature_potential[0] / R
    elif mode != "none":
        ref = cfg.get_real("method", "reference")
    t0 = time.perf_counter()
    rad = center / np.linalg.norm(center)
    exterior = scene.side == DomainSide.Exterior
    axis = rad if exterior else -rad
    theta_max = math.acos((-1.0 if exterior else 1.0) * a / (2.0 * R))
    dirs, wts = gamma_rule(nt, nphi, theta_max)
    est, _ = wos_patch_nodes(scene, w, center[None], axis[None], a, dirs)
    P = np.zeros(1, PATCH_DTYPE)
    P["o"], P["axis"], P["a"], P["R"], P["surf"] = center, axis, a, R, 0
    f = solve_patch(scene, P, dirs, wts, est, dcfg)
    rec.schema = "biewos_patch/v1"
    rec.columns = ["panel", "r", "dudn", "est_err", "ref", "err_pct"]
    for i in range(dcfg.m):
        rec.rows.append([i, f.r[0, i], f.dudn[0, i], f.est_error[0, i], _nan(ref),
                         _err_pct(f.dudn[0, i], ref)])
    rec.paths_total = float(nt) * nphi * w.n_paths
    rec.row_seconds.append(time.perf_counter() - t0)


def _run_dtn(cfg, rec, seed):
    """biewos_dtn: whole-boundary Neumann data of a BASELINE configuration."""
    from .dtn import BIE_FIRST, BIE_SECOND, DtnConfig, dtn_solve_workload
    from .workloads import CONFIGS

    kind_s = cfg.get_str("method", "kind", "second")  # runner.cpp:192-193
    if kind_s not in ("first", "second"):
        cfg.fail("method", "kind", f"expected first or second, got '{kind_s}'")
    dcfg = DtnConfig(kind=BIE_FIRST if kind_s == "first" else BIE_SECOND)
    c = cfg.get_int("method", "baseline_config", 1)
    n_bp = cfg.get_int("method", "n_bp", 0)
    w = CONFIGS[c]()
    if n_bp and n_bp < w.n_bp:
        w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, n_bp).astype(np.int64)))
    if seed is not None:
        w.seed = seed
    t0 = time.perf_counter()
    devices = _devices(cfg)
    if devices is None:
        res = dtn_solve_workload(w, dcfg, n_paths=cfg.get_int("method", "n_path", w.n_paths))
    else:  # the same bits on any device list (bw_group_dtn_solve)
        from .dtn import patches_for
        from .group import DeviceGroup

        g = DeviceGroup(devices)
        res, _, _ = g.dtn_solve(w.scene, w.wos_config(cfg.get_int("method", "n_path", w.n_paths)),
                                patches_for(w), w.dirs, w.weights, dcfg)
        g.close()
    exact = w.exact_dudn_outward()
    rec.schema = "biewos_dtn/v1"
    rec.columns = ["point", "x", "y", "z", "a", "dudn", "est_err", "ref", "err_pct", "status"]
    for i in range(w.n_bp):
        rec.rows.append([i, *w.points[i], w.radii[i], res.dudn[i], res.err[i], exact[i],
                         _err_pct(res.dudn[i], exact[i]), res.status[i]])
    rec.paths_total = float(w.n_bp) * w.n_nodes * cfg.get_int("method", "n_path", w.n_paths)
    rec.row_seconds.append(time.perf_counter() - t0)


def _devices(cfg):
    """[gpu] devices: device ids for the in-library device group;
    absent = the process's single context."""
    if not cfg.has("gpu", "devices"):
        return None
    return [int(float(t)) for t in cfg.tokens("gpu", "devices") if t != ";"]


def _run_pipeline(cfg, rec, seed):
    """biewos_pipeline: BASELINE config 5 — the DtN of every boundary point,
    the NCCL all-gather of the panel records and the integral representation
    (field_eval.cpp:7-19) at the targets, through bw_group_pipeline. Rows in
    the schema of the reference's field_eval method (runner.cpp:243-299): one
    per target, with the analytic potential as the reference column."""
    from .group import DeviceGroup
    from .pipeline import panel_areas
    from .dtn import DtnConfig, patches_for
    from .workloads import CONFIGS, make_targets

    c = cfg.get_int("method", "baseline_config", 5)
    if c not in (3, 5):
        cfg.fail("method", "baseline_config", "the pipeline needs a cavity-box configuration (3 or 5)")
    w = CONFIGS[c]()
    n_bp = cfg.get_int("method", "n_bp", 0)
    if n_bp and n_bp < w.n_bp:
        w = w.subset(np.unique(np.linspace(0, w.n_bp - 1, n_bp).astype(np.int64)))
    if seed is not None:
        w.seed = seed
    n_t = cfg.get_int("method", "n_targets", int(w.extra.get("n_targets", 1000000)))
    rng_s = cfg.get_str("method", "rng", "philox4x64")
    if rng_s not in ("philox4x64", "philox4x32"):
        cfg.fail("method", "rng", f"expected philox4x64 or philox4x32, got '{rng_s}'")
    targets = make_targets(w, n_t, seed=cfg.get_int("method", "target_seed", 5))
    wcfg = w.wos_config(cfg.get_int("method", "n_path", w.n_paths), 1 if rng_s == "philox4x32" else 0)
    t0 = time.perf_counter()
    g = DeviceGroup(_devices(cfg) or [0])
    r = g.pipeline(w.scene, wcfg, patches_for(w), w.dirs, w.weights, panel_areas(w),
                   np.asarray(w.scene.phi(w.points), np.float64), targets, DtnConfig())
    g.close()
    exact = w.exact_u(targets)
    rec.schema = "biewos_pipeline/v1"
    rec.columns = ["target", "tx", "ty", "tz", "u", "ref", "err_pct", "near"]
    for i in range(n_t):
        rec.rows.append([i, *targets[i], r.u[i], exact[i],
                         math.nan if r.near[i] else _err_pct(r.u[i], exact[i]), int(r.near[i])])
    rec.paths_total = float(w.n_bp) * w.n_nodes * wcfg.n_paths
    rec.row_seconds.append(time.perf_counter() - t0)


def _fmt(v) -> str:
    return "%.12g" % float(v)


def run(cfg: RawConfig, seed=None, workers=None) -> RunRecord:  # runner.cpp:345-390
    t_all = time.perf_counter()
    rec = RunRecord(method=cfg.get_str("method", "name"))
    if rec.method == "biewos_dtn":
        _run_dtn(cfg, rec, seed)
    elif rec.method == "biewos_pipeline":
        _run_pipeline(cfg, rec, seed)
    else:
        scene = scene_from_config(cfg)
        if rec.method == "biewos_point":
            _run_point(cfg, scene, rec, seed, workers)
        elif rec.method == "last_passage":
            _run_lp(cfg, scene, rec, seed, workers)
        elif rec.method == "field_eval":
            _run_field_eval(cfg, scene, rec)
        elif rec.method == "biewos_patch":
            _run_patch(cfg, scene, rec, seed)
        elif rec.method == "reference_bem":
            raise ApplicabilityError(f"method '{rec.method}' is not on the B200 path")
        else:
            cfg.fail("method", "name", f"unknown method '{rec.method}'")
    rec.wall_seconds = time.perf_counter() - t_all
    lines = [f"# biewos-csv schema={rec.schema}", f"# config: {cfg.echo()}", ",".join(rec.columns)]
    lines += [",".join(_fmt(v) for v in row) for row in rec.rows]
    rec.csv_text = "\n".join(lines) + "\n"
    rec.json_text = json.dumps({
        "version": VERSION, "method": rec.method, "schema": rec.schema, "config": cfg.echo(),
        "columns": rec.columns, "rows": [[float(v) for v in r] for r in rec.rows],
        "paths_total": rec.paths_total, "wall_seconds": rec.wall_seconds,
        "row_seconds": rec.row_seconds}, indent=2) + "\n"
    return rec


def write_outputs(rec: RunRecord, cfg: RawConfig) -> None:
    for key, text in (("csv", rec.csv_text), ("json", rec.json_text)):
        if cfg.has("output", key):
            path = cfg.get_str("output", key)
            try:
                with open(path, "w", newline="") as f:
                    f.write(text)
            except OSError:
                raise ConfigError(f"cannot write {key.upper()} output: {path}")


def _read_csv(path):
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise ConfigError(f"cannot open CSV file: {path}")
    rows = [ln.rstrip("\r").split(",") for ln in lines if ln and not ln.startswith("#")]
    return rows[0], rows[1:]


def compare_csv(file_a: str, file_b: str, tol: float, report=None) -> int:  # runner.cpp:445-479
    ca, ra = _read_csv(file_a)
    cb, rb = _read_csv(file_b)
    say = report.write if report is not None else (lambda s: None)
    if ca != cb:
        raise ConfigError(f"CSV schema mismatch between {file_a} and {file_b}")
    if len(ra) != len(rb):
        say(f"row count mismatch: {len(ra)} vs {len(rb)}\n")
        return 1
    fails = 0
    for r, (x, y) in enumerate(zip(ra, rb)):
        if len(x) != len(y):
            say(f"row {r}: cell count mismatch\n")
            fails += 1
            continue
        for c, (s, t) in enumerate(zip(x, y)):
            va, vb = float(s), float(t)
            if math.isnan(va) and math.isnan(vb):
                continue
            denom = max(abs(va), abs(vb))
            if abs(va - vb) > tol * denom:
                say(f"row {r} col {ca[c]}: {s} vs {t}\n")
                fails += 1
    say(f"compare: {'PASS' if not fails else 'FAIL'} ({len(ra)} rows, tol {tol})\n")
    return 0 if not fails else 1
