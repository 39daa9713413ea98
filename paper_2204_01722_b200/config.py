"""ProblemConfig and its key = value parser (config.hpp:28-273), and the
FemProblem wiring of a parsed config (problem.hpp:19-58, :81-127).

Same keys, defaults, value syntax and error messages as the reference
(ConfigError, errors.hpp:83-99), so a reference config file drives this
framework unchanged.  `threads` and `deterministic` are accepted and
ignored (the device path is deterministic by construction)."""
from __future__ import annotations

import dataclasses
import io
from dataclasses import dataclass, field

FACE_NAMES = ("-x", "+x", "-y", "+y", "-z", "+z")


class ConfigError(ValueError):
    """errors.hpp:83-99: 'config line L (key 'k'): msg' or 'config: msg'."""

    def __init__(self, msg, line=0, key=""):
        text = (f"config line {line}" + (f" (key '{key}')" if key else "") + f": {msg}"
                if line > 0 else f"config: {msg}")
        super().__init__(text)
        self.line, self.key = line, key


@dataclass(frozen=True)
class StudyCase:
    """One (order, refinement) study case, parsed from 'PxR' (config.hpp:17-26)."""
    order: int = 1
    refinement: int = 1

    def id(self):
        return f"p{self.order}r{self.refinement}"


@dataclass
class ProblemConfig:
    """config.hpp:28-86; every field has the reference's default."""
    case_id: str = "case"
    extents: list = field(default_factory=lambda: [1.0, 1.0, 1.0])
    cells: list = field(default_factory=lambda: [1, 1, 1])
    order: int = 2
    geometry_order: int = 0
    quadrature_points: int = 0
    youngs_modulus: float = 1.0
    poisson_ratio: float = 0.3
    mu: float = 0.0
    lam: float = 0.0
    storage: str = "current"
    fixed_faces: list = field(default_factory=lambda: ["-x"])
    traction_face: str = "none"
    traction: list = field(default_factory=lambda: [0.0, 0.0, 0.0])
    body_force: list = field(default_factory=lambda: [0.0, 0.0, 0.0])
    solver: str = "newton-cg"
    load_steps: int = 1
    newton_rtol: float = 1e-8
    newton_atol: float = 1e-10
    newton_max_iterations: int = 50
    linear_rtol: float = 1e-3
    linear_max_iterations: int = 500
    line_search: bool = True
    lbfgs_memory: int = 5
    precond_refresh: int = 10
    mg_pre_smooth: int = 1
    mg_post_smooth: int = 1
    threads: int = 1
    deterministic: bool = False
    write_vtk: bool = False
    study_cases: list = field(default_factory=list)
    study_reference: StudyCase = StudyCase(3, 3)
    perf_orders: list = field(default_factory=lambda: [1, 2, 3])
    perf_target_dofs: list = field(default_factory=lambda: [3000, 20000])
    perf_representations: list = field(default_factory=lambda: ["matrix-free", "assembled"])
    perf_repeats: int = 20

    def material(self):
        """(mu, lambda): explicit when mu is set, else from Young/Poisson (config.hpp:82-85)."""
        if self.mu != 0.0:
            return self.mu, self.lam
        E, nu = self.youngs_modulus, self.poisson_ratio
        return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))

    def copy(self, **changes):
        return dataclasses.replace(self, **changes)


def _number(v, line, key, kind):
    try:
        if kind is int:
            if v.strip() != v or not v or not (v.lstrip("+-").isdigit()):
                raise ValueError
            return int(v)
        return float(v)
    except ValueError:
        raise ConfigError(f"expected {'an integer' if kind is int else 'a number'}, got '{v}'",
                          line, key) from None


def _bool(v, line, key):
    if v in ("true", "1", "yes", "on"):
        return True
    if v in ("false", "0", "no", "off"):
        return False
    raise ConfigError(f"expected a boolean, got '{v}'", line, key)


def _face(v, line, key):
    if v not in FACE_NAMES:
        raise ConfigError(f"expected a face (+x -x +y -y +z -z), got '{v}'", line, key)
    return v


def _case(tok, line, key):
    if "x" not in tok:
        raise ConfigError(f"expected ORDERxREFINEMENT, got '{tok}'", line, key)
    a, b = tok.split("x", 1)
    c = StudyCase(_number(a, line, key, int), _number(b, line, key, int))
    if c.order < 1 or c.refinement < 1:
        raise ConfigError(f"case '{tok}' must have order and refinement >= 1", line, key)
    return c


_SCALARS = {
    "case_id": ("case_id", str), "order": ("order", int), "geometry_order": ("geometry_order", int),
    "quadrature_points": ("quadrature_points", int), "youngs_modulus": ("youngs_modulus", float),
    "poisson_ratio": ("poisson_ratio", float), "mu": ("mu", float), "lambda": ("lam", float),
    "load_steps": ("load_steps", int), "newton_rtol": ("newton_rtol", float),
    "newton_atol": ("newton_atol", float), "newton_max_iterations": ("newton_max_iterations", int),
    "linear_rtol": ("linear_rtol", float), "linear_max_iterations": ("linear_max_iterations", int),
    "lbfgs_memory": ("lbfgs_memory", int), "precond_refresh": ("precond_refresh", int),
    "mg_pre_smooth": ("mg_pre_smooth", int), "mg_post_smooth": ("mg_post_smooth", int),
    "threads": ("threads", int), "perf_repeats": ("perf_repeats", int),
}
_VEC = {"length_": "extents", "cells_": "cells", "traction_": "traction", "body_force_": "body_force"}


def parse_problem_config(text_or_stream) -> ProblemConfig:
    """parse_problem_config (config.hpp:164-262): '#' comments, 'key = value'
    lines, unknown keys rejected."""
    stream = io.StringIO(text_or_stream) if isinstance(text_or_stream, str) else text_or_stream
    cfg = ProblemConfig()
    for line_no, raw in enumerate(stream, start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError("expected 'key = value'", line_no, line)
        key, value = (t.strip() for t in line.split("=", 1))
        if not key:
            raise ConfigError("empty key", line_no)
        if key in _SCALARS:
            attr, kind = _SCALARS[key]
            setattr(cfg, attr, value if kind is str else _number(value, line_no, key, kind))
            continue
        vec = next((p for p in _VEC if key.startswith(p) and key[len(p):] in ("x", "y", "z")), None)
        if vec is not None:
            d = "xyz".index(key[len(vec):])
            kind = int if vec == "cells_" else float
            getattr(cfg, _VEC[vec])[d] = _number(value, line_no, key, kind)
            continue
        if key == "jacobian_storage":
            if value not in ("current", "initial-native", "initial-tuned", "initial-ad"):
                raise ConfigError(f"unknown jacobian storage '{value}'", line_no, key)
            cfg.storage = value
        elif key == "fixed_faces":
            cfg.fixed_faces = [_face(t, line_no, key) for t in value.split()]
        elif key == "traction_face":
            if value != "none":
                _face(value, line_no, key)
            cfg.traction_face = value
        elif key == "solver":
            if value not in ("newton-cg", "lbfgs"):
                raise ConfigError(f"unknown solver '{value}'", line_no, key)
            cfg.solver = value
        elif key == "line_search":
            if value not in ("critical-point", "none"):
                raise ConfigError(f"unknown line search '{value}'", line_no, key)
            cfg.line_search = value == "critical-point"
        elif key in ("deterministic", "write_vtk"):
            setattr(cfg, key, _bool(value, line_no, key))
        elif key == "study_cases":
            cfg.study_cases = [_case(t, line_no, key) for t in value.split()]
        elif key == "study_reference":
            cfg.study_reference = _case(value, line_no, key)
        elif key == "perf_orders":
            cfg.perf_orders = [_number(t, line_no, key, int) for t in value.split()]
        elif key == "perf_target_dofs":
            cfg.perf_target_dofs = [_number(t, line_no, key, int) for t in value.split()]
        elif key == "perf_representations":
            toks = value.split()
            for t in toks:
                if t not in ("matrix-free", "assembled"):
                    raise ConfigError(f"unknown representation '{t}'", line_no, key)
            cfg.perf_representations = toks
        else:
            raise ConfigError("unknown key", line_no, key)
    return cfg


def load_problem_config(path) -> ProblemConfig:
    """load_problem_config (config.hpp:264-268)."""
    try:
        with open(path) as f:
            return parse_problem_config(f)
    except OSError:
        raise OSError(f"cannot open config file '{path}'") from None


def newton_overrides(cfg: ProblemConfig, reference_line_search_quirk=False) -> dict:
    """FemProblem::newton_config + sanitize (problem.hpp:97-108, :130-136).
    reference_line_search_quirk reproduces the reference's post-line-search
    residual defect for byte-level comparisons."""
    if (cfg.newton_max_iterations < 1 or cfg.newton_rtol <= 0 or cfg.newton_atol <= 0
            or cfg.linear_rtol <= 0 or cfg.load_steps < 1):
        raise ConfigError("solver tolerances must be positive and counts >= 1")
    return dict(max_iterations=cfg.newton_max_iterations, rtol=cfg.newton_rtol,
                atol=cfg.newton_atol, linear_rtol=cfg.linear_rtol,
                linear_max_iterations=cfg.linear_max_iterations,
                use_line_search=int(cfg.line_search), load_steps=cfg.load_steps,
                solver=1 if cfg.solver == "lbfgs" else 0, lbfgs_memory=cfg.lbfgs_memory,
                precond_refresh=cfg.precond_refresh,
                reference_line_search_quirk=int(reference_line_search_quirk))


def build_problem(cfg: ProblemConfig):
    """FemProblem(cfg) (problem.hpp:19-58) on the device."""
    from .hexmg import FemProblem
    if cfg.order < 1:
        raise ConfigError("order must be >= 1")
    mu, lam = cfg.material()
    return FemProblem(extents=tuple(cfg.extents), cells=tuple(cfg.cells), order=cfg.order,
                      q=cfg.quadrature_points, fixed_faces=tuple(cfg.fixed_faces),
                      traction_face=None if cfg.traction_face == "none" else cfg.traction_face,
                      traction=tuple(cfg.traction), body_force=tuple(cfg.body_force),
                      mu=mu, lam=lam, storage=cfg.storage,
                      mg_smoothing=(cfg.mg_pre_smooth, cfg.mg_post_smooth))
