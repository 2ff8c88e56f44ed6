"""Generate tests/golden/templates_golden.json: canonical JSON of every reference fixture,
parsed by the REFERENCE loaders (/root/reference/pkg/src/batchsim/assets.py).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_template_golden.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_pose_golden import load_reference  # noqa: E402


def main():
    load_reference()
    import batchsim_ref.assets as A
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "batchsim_ref_fixtures", "/root/reference/pkg/src/batchsim/tasks/fixtures.py")
    F = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(F)
    out = {}
    for name in ("PENDULUM_URDF", "LONG_PENDULUM_URDF", "PLANAR_2R_URDF", "ARM3_URDF",
                 "PUSHER_XY_URDF", "PEN_XYZ_URDF"):
        out[name] = A.load_urdf(getattr(F, name)).to_dict()
    out["CARTPOLE_MJCF"] = [t.to_dict() for t in A.load_mjcf(F.CARTPOLE_MJCF)]
    for d in (1, 2, 3, 5, 6):
        out[f"chain{d}"] = A.load_urdf(F.make_chain_urdf(d)).to_dict()
    path = os.path.join(HERE, "templates_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, sort_keys=True, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
