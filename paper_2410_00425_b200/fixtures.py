"""Primitive-only robot fixtures for the task suite, generated from compact specs.

Same robots as the reference fixtures (``/root/reference/pkg/src/batchsim/tasks/fixtures.py``
:8-296): the parsed templates are canonical-JSON equal to the reference's
(tests/test_assets.py).  Here they are emitted by a small URDF writer instead of being
stored as literal XML, plus one fixture the reference lacks: the synthetic cabinet family
used by the articulated-object config (decision A-18).
"""

from __future__ import annotations

HALF_PI = "1.5707963267948966"


def _inertial(mass, diag, xyz=None):
    org = f'\n      <origin xyz="{xyz}"/>' if xyz else ""
    ixx, iyy, izz = diag
    return (f"    <inertial>{org}\n      <mass value=\"{mass}\"/>\n"
            f"      <inertia ixx=\"{ixx}\" ixy=\"0\" ixz=\"0\" iyy=\"{iyy}\" iyz=\"0\" izz=\"{izz}\"/>\n"
            f"    </inertial>")


def _collision(geom, xyz=None, rpy=None):
    attrs = ""
    if xyz or rpy:
        attrs = "\n      <origin" + (f' xyz="{xyz}"' if xyz else "") + (f' rpy="{rpy}"' if rpy else "") + "/>"
    return f"    <collision>{attrs}\n      <geometry>{geom}</geometry>\n    </collision>"


def _link(name, *parts, color=None):
    body = [p for p in parts if p]
    if color:
        body.append(f'    <visual><material><color rgba="{color}"/></material></visual>')
    if not body:
        return f'  <link name="{name}"/>'
    return f'  <link name="{name}">\n' + "\n".join(body) + "\n  </link>"


def _joint(name, jtype, parent, child, axis=None, xyz=None, limit=None, damping=None):
    rows = [f'  <joint name="{name}" type="{jtype}">']
    if xyz:
        rows.append(f'    <origin xyz="{xyz}"/>')
    rows += [f'    <parent link="{parent}"/>', f'    <child link="{child}"/>']
    if axis:
        rows.append(f'    <axis xyz="{axis}"/>')
    if limit:
        rows.append(f'    <limit lower="{limit[0]}" upper="{limit[1]}"/>')
    if damping is not None:
        rows.append(f'    <dynamics damping="{damping}"/>')
    rows.append("  </joint>")
    return "\n".join(rows)


def _robot(name, links, joints):
    return "\n".join(['<?xml version="1.0"?>', f'<robot name="{name}">', *links, *joints, "</robot>", ""])


def _capsule(r, length):
    return f'<capsule radius="{r}" length="{length}"/>'


def _pendulum(bob_z: str) -> str:
    return _robot("pendulum", [
        _link("base"),
        _link("bob", _inertial("1.0", ("0", "0", "0"), f"0 0 {bob_z}"),
              _collision('<sphere radius="0.05"/>', xyz=f"0 0 {bob_z}")),
    ], [_joint("swing", "continuous", "base", "bob", axis="0 1 0")])


PENDULUM_URDF = _pendulum("-1.0")
LONG_PENDULUM_URDF = _pendulum("-2.0")


def _planar_2r() -> str:
    arm = lambda n: _link(n, _inertial("1.0", ("0.001", "0.084", "0.084"), "0.5 0 0"),  # noqa: E731
                          _collision(_capsule("0.04", "0.9"), xyz="0.5 0 0", rpy=f"0 {HALF_PI} 0"))
    return _robot("planar_2r", [_link("base"), arm("upper"), arm("fore"), _link("tip")], [
        _joint("shoulder", "revolute", "base", "upper", axis="0 0 1", limit=("-3.1415", "3.1415")),
        _joint("elbow", "revolute", "upper", "fore", axis="0 0 1", xyz="1.0 0 0",
               limit=("-3.1415", "3.1415")),
        _joint("tip_weld", "fixed", "fore", "tip", xyz="1.0 0 0"),
    ])


PLANAR_2R_URDF = _planar_2r()


def _arm3() -> str:
    """3-DOF arm: yaw about z, shoulder/elbow about y, links along +x, ee sphere at 0.8 m."""
    seg = lambda n, m, iyy: _link(  # noqa: E731
        n, _inertial(m, ("0.001", iyy, iyy), "0.2 0 0"),
        _collision(_capsule("0.03", "0.32"), xyz="0.2 0 0", rpy=f"0 {HALF_PI} 0"))
    return _robot("arm3", [
        _link("root"),
        _link("shoulder_link", _inertial("0.5", ("0.002", "0.002", "0.002"))),
        seg("upper_arm", "0.8", "0.012"),
        seg("forearm", "0.6", "0.009"),
        _link("ee", _inertial("0.1", ("0.0001", "0.0001", "0.0001")),
              _collision('<sphere radius="0.03"/>'), color="0.9 0.2 0.2 1"),
    ], [
        _joint("yaw", "revolute", "root", "shoulder_link", axis="0 0 1", limit=("-3.1", "3.1"), damping="0.1"),
        _joint("shoulder", "revolute", "shoulder_link", "upper_arm", axis="0 1 0", limit=("-2.2", "2.2"),
               damping="0.1"),
        _joint("elbow", "revolute", "upper_arm", "forearm", axis="0 1 0", xyz="0.4 0 0",
               limit=("-2.4", "2.4"), damping="0.1"),
        _joint("ee_weld", "fixed", "forearm", "ee", xyz="0.4 0 0"),
    ])


ARM3_URDF = _arm3()


def make_arm6_urdf(name: str = "arm6") -> str:
    """6-DOF arm for the full-twist pd_ee_delta_pose KAT ("a reachable arm"): ARM3's
    yaw / shoulder / elbow and links, then a spherical wrist at the forearm tip (roll about x,
    pitch about y, roll about x; concentric axes) and the ee sphere 0.1 m beyond it.  A 3-DOF
    arm cannot follow a 6-D twist (DLS trades the rotation rows); this one can."""
    seg = lambda n, m, iyy: _link(  # noqa: E731
        n, _inertial(m, ("0.001", iyy, iyy), "0.2 0 0"),
        _collision(_capsule("0.03", "0.32"), xyz="0.2 0 0", rpy=f"0 {HALF_PI} 0"))
    small = lambda n: _link(n, _inertial("0.1", ("0.0002", "0.0002", "0.0002")))  # noqa: E731
    return _robot(name, [
        _link("root"),
        _link("shoulder_link", _inertial("0.5", ("0.002", "0.002", "0.002"))),
        seg("upper_arm", "0.8", "0.012"),
        seg("forearm", "0.6", "0.009"),
        small("wrist_roll_link"),
        small("wrist_pitch_link"),
        _link("hand", _inertial("0.1", ("0.0002", "0.0002", "0.0002"), "0.05 0 0")),
        _link("ee", _inertial("0.05", ("0.0001", "0.0001", "0.0001")),
              _collision('<sphere radius="0.03"/>'), color="0.9 0.2 0.2 1"),
    ], [
        _joint("yaw", "revolute", "root", "shoulder_link", axis="0 0 1", limit=("-3.1", "3.1"), damping="0.1"),
        _joint("shoulder", "revolute", "shoulder_link", "upper_arm", axis="0 1 0", limit=("-2.2", "2.2"),
               damping="0.1"),
        _joint("elbow", "revolute", "upper_arm", "forearm", axis="0 1 0", xyz="0.4 0 0",
               limit=("-2.4", "2.4"), damping="0.1"),
        _joint("wrist_roll", "revolute", "forearm", "wrist_roll_link", axis="1 0 0", xyz="0.4 0 0",
               limit=("-3.1", "3.1"), damping="0.05"),
        _joint("wrist_pitch", "revolute", "wrist_roll_link", "wrist_pitch_link", axis="0 1 0",
               limit=("-2.0", "2.0"), damping="0.05"),
        _joint("wrist_roll2", "revolute", "wrist_pitch_link", "hand", axis="1 0 0", limit=("-3.1", "3.1"),
               damping="0.05"),
        _joint("ee_weld", "fixed", "hand", "ee", xyz="0.1 0 0"),
    ])


ARM6_URDF = make_arm6_urdf()


def _gantry(name, carriages, tip, axes, limits, tip_shape=None, tip_color=None):
    links = [_link("frame")]
    for cname, mass, inert in carriages:
        links.append(_link(cname, _inertial(mass, (inert, inert, inert))))
    tname, tmass, tinert = tip
    links.append(_link(tname, _inertial(tmass, (tinert, tinert, tinert)),
                       _collision(tip_shape) if tip_shape else None, color=tip_color))
    chain = ["frame"] + [c[0] for c in carriages] + [tname]
    joints = [_joint(f"slide_{ax}", "prismatic", chain[i], chain[i + 1], axis=vec, limit=lim, damping="1.0")
              for i, (ax, vec, lim) in enumerate(zip("xyz", axes, limits))]
    return _robot(name, links, joints)


PUSHER_XY_URDF = _gantry("pusher_xy", [("carriage_x", "0.5", "0.001")], ("tip", "0.3", "0.0005"),
                         ["1 0 0", "0 1 0"], [("-0.6", "0.6")] * 2, '<sphere radius="0.03"/>',
                         "0.2 0.8 0.3 1")
PEN_XYZ_URDF = _gantry("pen_xyz", [("carriage_x", "0.4", "0.001"), ("carriage_y", "0.4", "0.001")],
                       ("pen_tip", "0.2", "0.0004"), ["1 0 0", "0 1 0", "0 0 1"],
                       [("-0.5", "0.5"), ("-0.5", "0.5"), ("0.0", "0.4")], None, "0.1 0.1 0.1 1")

CARTPOLE_MJCF = """<?xml version="1.0"?>
<mujoco model="cartpole">
  <compiler angle="radian"/>
  <default>
    <joint damping="0.0"/>
    <default class="viz"><geom rgba="0.3 0.5 0.9 1"/></default>
  </default>
  <worldbody>
    <body name="cart" pos="0 0 0.1">
      <joint name="slider" type="slide" axis="1 0 0" range="-1.8 1.8"/>
      <inertial pos="0 0 0" mass="1.0" diaginertia="0.004 0.004 0.004"/>
      <geom name="cart_geom" type="box" size="0.1 0.05 0.05" class="viz"/>
      <body name="pole" pos="0 0 0">
        <joint name="hinge" type="hinge" axis="0 1 0"/>
        <inertial pos="0 0 0.3" mass="0.1" diaginertia="0.003 0.003 0.00001"/>
        <geom name="pole_geom" type="capsule" size="0.02 0.3" pos="0 0 0.3" rgba="0.9 0.6 0.2 1"/>
      </body>
    </body>
  </worldbody>
</mujoco>
"""


def make_chain_urdf(dof: int, link_length: float = 0.3, name: str = "chain") -> str:
    """Serial revolute chain along +x with alternating z/y axes (fixtures.py:263-296)."""
    if dof < 1:
        raise ValueError("chain needs at least 1 DOF")
    links, joints = [_link("base")], []
    half = link_length / 2
    for i in range(dof):
        links.append(_link(f"link{i}", _inertial("0.5", ("0.0005", "0.004", "0.004"), f"{half} 0 0"),
                           _collision(_capsule("0.02", f"{link_length * 0.9}"), xyz=f"{half} 0 0",
                                      rpy=f"0 {HALF_PI} 0")))
        joints.append(_joint(f"joint{i}", "revolute", "base" if i == 0 else f"link{i - 1}", f"link{i}",
                             axis="0 0 1" if i % 2 == 0 else "0 1 0",
                             xyz="0 0 0" if i == 0 else f"{link_length} 0 0", limit=("-1.2", "1.2"),
                             damping="0.05"))
    return _robot(f"{name}{dof}", links, joints)


def make_cabinet_urdf(kinds: str, name: str = "cabinet") -> str:
    """Synthetic cabinet (decision A-18): a fixed box carcass with one articulated part per
    character of ``kinds`` -- 'd' = prismatic drawer (slides +x out of the front face),
    'r' = revolute door (hinged about z at the front-left edge).  Parts stack vertically.
    Box links only (box/box contact is outside the supported pair set, so the
    parts are held by joint limits, not contacts)."""
    if not 1 <= len(kinds) <= 6 or set(kinds) - set("dr"):
        raise ValueError("kinds must be 1-6 characters of 'd'/'r'")
    n = len(kinds)
    slot_h = 0.1
    height = n * slot_h
    links = [_link("carcass", _inertial("5.0", ("0.1", "0.1", "0.1")),
                   _collision(f'<box size="0.3 0.4 {height:.3f}"/>', xyz=f"0 0 {height / 2:.3f}"),
                   color="0.55 0.4 0.25 1")]
    joints = []
    for i, k in enumerate(kinds):
        zc = slot_h * i + slot_h / 2
        if k == "d":
            links.append(_link(f"drawer{i}", _inertial("0.4", ("0.002", "0.002", "0.002")),
                               _collision('<box size="0.28 0.36 0.08"/>', xyz="-0.14 0 0"),
                               color="0.8 0.7 0.5 1"))
            joints.append(_joint(f"drawer{i}_joint", "prismatic", "carcass", f"drawer{i}", axis="1 0 0",
                                 xyz=f"0.15 0 {zc:.3f}", limit=("0", "0.25"), damping="1.0"))
        else:
            links.append(_link(f"door{i}", _inertial("0.3", ("0.002", "0.002", "0.002"), "0 -0.19 0"),
                               _collision('<box size="0.02 0.38 0.09"/>', xyz="0 -0.19 0"),
                               color="0.7 0.5 0.35 1"))
            joints.append(_joint(f"door{i}_joint", "revolute", "carcass", f"door{i}", axis="0 0 1",
                                 xyz=f"0.16 0.2 {zc:.3f}", limit=("0", "1.5"), damping="0.5"))
    return _robot(name, links, joints)


def make_mobile_base_urdf(name: str = "mobile_base") -> str:
    """Abstract mobile base for the ``base_forward_rotate`` controller (PAPER §A.2:
    "one joint controlling forward/backward movement and another controlling rotation"):
    world-fixed root -> prismatic x -> prismatic y -> revolute yaw -> box chassis.  The
    controller drives the planar joints kinematically from (forward speed, yaw rate)."""
    links = [_link("odom"),
             _link("base_x", _inertial("5.0", ("0.05", "0.05", "0.05"))),
             _link("base_y", _inertial("5.0", ("0.05", "0.05", "0.05"))),
             _link("chassis", _inertial("10.0", ("0.2", "0.3", "0.4")),
                   _collision('<box size="0.5 0.4 0.2"/>', xyz="0 0 0.3"), color="0.3 0.3 0.35 1")]
    joints = [_joint("base_x_joint", "prismatic", "odom", "base_x", axis="1 0 0", limit=("-5", "5"), damping="1.0"),
              _joint("base_y_joint", "prismatic", "base_x", "base_y", axis="0 1 0", limit=("-5", "5"), damping="1.0"),
              _joint("base_yaw_joint", "revolute", "base_y", "chassis", axis="0 0 1", limit=("-1e9", "1e9"),
                     damping="1.0")]
    return _robot(name, links, joints)
