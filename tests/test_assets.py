"""Host-side robot-description loaders: templates equal the reference's (canonical JSON),
plus the SPEC's loader examples and error paths."""

import json
import math
import os

import pytest

from paper_2410_00425_b200 import assets as A
from paper_2410_00425_b200 import fixtures as F
from paper_2410_00425_b200.errors import AssetParseError, SchemaError, TopologyError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "templates_golden.json")))


@pytest.mark.parametrize("name", ["PENDULUM_URDF", "LONG_PENDULUM_URDF", "PLANAR_2R_URDF",
                                  "ARM3_URDF", "PUSHER_XY_URDF", "PEN_XYZ_URDF"])
def test_urdf_fixtures_match_reference(name):
    assert A.load_urdf(getattr(F, name)).to_dict() == GOLD[name]


def test_mjcf_cartpole_matches_reference():
    assert [t.to_dict() for t in A.load_mjcf(F.CARTPOLE_MJCF)] == GOLD["CARTPOLE_MJCF"]


@pytest.mark.parametrize("dof", [1, 2, 3, 5, 6])
def test_chain_matches_reference(dof):
    assert A.load_urdf(F.make_chain_urdf(dof)).to_dict() == GOLD[f"chain{dof}"]


def test_spec_examples():
    t = A.load_urdf(F.PLANAR_2R_URDF)
    assert t.dof == 2 and [l.name for l in t.links][:3] == ["base", "upper", "fore"]
    single = A.load_urdf('<robot name="r"><link name="only"/></robot>')
    assert single.dof == 0 and len(single.links) == 1
    with pytest.raises(SchemaError):
        A.load_urdf('<robot name="r"><link name="a"/><joint name="j" type="fixed">'
                    '<parent link="a"/><child link="ghost"/></joint></robot>')
    (cp,) = A.load_mjcf(F.CARTPOLE_MJCF)
    assert cp.dof == 2 and [j.joint_type for j in cp.movable_joints] == ["prismatic", "revolute"]
    two = A.load_mjcf('<mujoco><worldbody><body name="a"><geom size="0.1"/></body>'
                      '<body name="b"><geom size="0.1"/></body></worldbody></mujoco>')
    assert len(two) == 2
    dflt = A.load_mjcf('<mujoco><default><geom type="box" size="0.1 0.2 0.3"/></default>'
                       '<worldbody><body name="a"><geom/></body></worldbody></mujoco>')
    assert dflt[0].links[0].collision_shapes[0].size == (0.1, 0.2, 0.3)


def test_error_paths():
    with pytest.raises(AssetParseError, match="line"):
        A.load_urdf("<robot><link name='a'></robot>")
    with pytest.raises(TopologyError):
        A.load_urdf('<robot><link name="a"/><link name="b"/></robot>')
    with pytest.raises(SchemaError):
        A.load_urdf('<robot><link name="a"/><link name="b"/><joint name="j" type="planar">'
                    '<parent link="a"/><child link="b"/></joint></robot>')
    with pytest.raises(SchemaError):
        A.load_mjcf('<mujoco><worldbody><body name="a"><joint type="ball"/><geom size="1"/>'
                    '</body></worldbody></mujoco>')


def test_round_trip_and_defaults():
    t = A.load_urdf(F.ARM3_URDF)
    assert A.ArticulationTemplate.from_json(t.to_json()) == t
    assert t.joint_by_name("elbow").origin.pos == (0.4, 0.0, 0.0)
    assert math.isinf(A.load_urdf(F.PENDULUM_URDF).joints[0].limits[1])


@pytest.mark.parametrize("kinds", ["d", "rr", "drd", "dddddd", "rdrdrd"])
def test_cabinet_family(kinds):
    t = A.load_urdf(F.make_cabinet_urdf(kinds))
    assert t.dof == len(kinds)
    assert [j.joint_type for j in t.joints] == ["prismatic" if k == "d" else "revolute" for k in kinds]


def test_mobile_base_fixture():
    t = A.load_urdf(F.make_mobile_base_urdf())
    assert t.dof == 3
    assert [j.joint_type for j in t.joints] == ["prismatic", "prismatic", "revolute"]
