"""Scene configuration (TOML schema + build_scene), 2D and 3D."""
from .config import (SCHEMA, SceneConfig, SceneParseError, SceneValidationError, build_scene,
                     load_scene, set_fields, taylor_green_fn, validate_scene)

__all__ = ["SCHEMA", "SceneConfig", "SceneParseError", "SceneValidationError", "build_scene",
           "load_scene", "set_fields", "taylor_green_fn", "validate_scene"]
