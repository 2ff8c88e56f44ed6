"""ctypes mirrors of the C-ABI structs in include/batchsim_b200.h (field order is ABI)."""

from __future__ import annotations

import ctypes

from . import _native

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
F64 = ctypes.c_double


class BsModelTables(ctypes.Structure):
    _fields_ = [(n, I32) for n in ("num_models", "L_max", "D_max", "S_max", "P_max", "A_max", "C_max")] + [
        (n, P) for n in (
            "n_links", "n_dof", "n_shapes", "n_pairs", "n_actors", "link_parent", "link_jtype", "link_dof",
            "link_grounded", "link_axis", "link_org", "link_mass", "link_com", "link_inertia", "dof_lower",
            "dof_upper", "dof_damping", "dof_kp", "dof_kd", "dof_flim", "dof_ctrl", "shape_btype", "shape_body",
            "shape_kind", "shape_seg", "shape_size", "shape_frame", "shape_radius", "shape_color", "pair_i",
            "pair_j", "pair_code", "pair_slot", "actor_mass", "actor_inertia", "actor_rest")] + [("A_dyn", I32)]


class BsEnvState(ctypes.Structure):
    _fields_ = [("num_envs", I32), ("env_offset", I64)] + [
        (n, P) for n in ("model_id", "qpos", "qvel", "target", "actor_pose", "actor_vel", "link_pose", "goal",
                         "diverged", "elapsed", "reset_count", "target_dof", "ep_return", "ep_flags")]


class BsStepOutputs(ctypes.Structure):
    _fields_ = [("obs", P), ("obs_dim", I32)] + [
        (n, P) for n in ("reward", "terminated", "truncated", "success", "fail", "unsupported_pairs",
                         "contact_count", "contact_pairs", "contact_geom", "ep_done", "ep_return_out",
                         "ep_length_out", "ep_flags_out", "final_obs")]


class BsSimParams(ctypes.Structure):
    _fields_ = [("dt", F64), ("substeps", I32), ("pos_iters", I32), ("vel_iters", I32),
                ("gravity", F64 * 3), ("friction", F64), ("beta", F64), ("slop", F64),
                ("ctrl_mode", I32), ("action_dim", I32), ("action_scale", F64), ("action_scale_rot", F64), ("ik_lambda", F64),
                ("ee_link", I32), ("task", I32), ("max_steps", I32), ("auto_reset", I32),
                ("early_termination", I32), ("seed", ctypes.c_uint64), ("task_f", F64 * 16),
                ("control_freq", F64)]


F32 = ctypes.c_float


class BsMeshTables(ctypes.Structure):
    _fields_ = [("num_models", I32), ("V_max", I32), ("T_max", I32)] + [
        (n, P) for n in ("n_verts", "n_tris", "verts", "vert_shape", "tris", "tri_shape", "tri_packed")]


class BsCameraBatch(ctypes.Structure):
    _fields_ = [("num_cams", I32), ("width", I32), ("height", I32), ("near_plane", F32), ("far_plane", F32),
                ("mount_link", P), ("pose", P), ("intrinsics", P)]


class BsRenderParams(ctypes.Structure):
    _fields_ = [("light_dir", F64 * 3), ("ambient", F32), ("diffuse", F32), ("background", F32 * 3),
                ("tile", I32), ("frame_scratch", P), ("frame_queue", P)]


class BsFrameBatch(ctypes.Structure):
    _fields_ = [(n, P) for n in ("rgb", "depth", "seg", "pointcloud")]


_R = ctypes.POINTER
_native.register("bs_step", [_R(BsModelTables), _R(BsEnvState), _R(BsStepOutputs), _R(BsSimParams), P, P])
_native.register("bs_debug_phase_clocks", [P, I32, I32])
_native.register("bs_reset", [_R(BsModelTables), _R(BsEnvState), _R(BsStepOutputs), _R(BsSimParams), P, I32, P])
_native.register("bs_forward_kinematics", [_R(BsModelTables), _R(BsEnvState), P])
_native.register("bs_random_actions", [ctypes.c_uint64, I64, I64, I32, I32, P, P])
_native.register("bs_masked_copy", [P, P, I64, I64, P, P])
_native.register("bs_voxelize", [P, I64, P, I64, I64, P, F32, I32, I32, I32, P, P])
_native.register("bs_composite_greenscreen", [P, P, P, I64, I64, I64, P, P])
_native.register("bs_render", [_R(BsModelTables), _R(BsEnvState), _R(BsMeshTables), _R(BsCameraBatch), P,
                               _R(BsRenderParams), _R(BsFrameBatch), P])

# enum values (include/batchsim_b200.h)
KIND = {"sphere": 0, "box": 1, "capsule": 2, "cylinder": 3, "plane": 4}
JOINT = {"fixed": 0, "revolute": 1, "prismatic": 2}
BODY_LINK, BODY_ACTOR, BODY_STATIC = 0, 1, 2
PAIR_CODE = {(0, 4): 1, (1, 4): 2, (0, 0): 3, (0, 1): 4, (2, 4): 5}
PAIR_MAXC = {1: 1, 2: 4, 3: 1, 4: 1, 5: 2}
PAIR_SWAP = 16
CTRL = {"pd_joint_pos": 0, "pd_joint_delta_pos": 1, "pd_ee_delta_pose": 2, "base_forward_rotate": 3}
TASK_NONE, TASK_PICKCUBE, TASK_OPENCHAIN, TASK_CARTPOLE = 0, 1, 2, 3
