"""Host logic of the shared face evaluation (no GPU): the role tables the
one-pass kernels are launched with (esdg_b200_face_roles, csrc/host/mesh.cpp).

The reference keeps ONE record per face and lets both sides read it
(compute_face_record / commit_face_side, kernels.hpp:350-430; its face list
has one entry per face, mesh.cpp:96-132). The GPU path gets the same "every
interior face is evaluated exactly once" from a per-element role byte: the
element on the minus side of a face evaluates it and pushes the other
element's lift term, which that element pulls. A pull may only depend on an
element that is dispatched no later in the same launch, or the launch could
wait on itself.
"""
import numpy as np
import pytest

from paper_2605_16684_b200 import capi

MESHES = [
    ("bubble walls+periodic", lambda: capi.bubble_mesh_config(2, False)),
    ("bubble periodic", lambda: capi.bubble_mesh_config(2, True)),
    ("two across", lambda: capi.bubble_mesh_config(1, True)),
    ("one element", lambda: capi.bubble_mesh_config(0, True)),
    ("channel", lambda: capi.channel_mesh_config(1, (3, 2, 1))),
]


def roles_of(mesh, world, rank, epb, split):
    h = capi.rank_halo(mesh, world, rank)
    return h, capi.face_roles(h["nbr_local"], epb, split)


@pytest.mark.parametrize("name,cfg", MESHES, ids=[m[0] for m in MESHES])
@pytest.mark.parametrize("epb", [1, 5, 8])
@pytest.mark.parametrize("world", [1, 3])
@pytest.mark.parametrize("split", [False, True])
def test_every_local_face_has_one_evaluator(name, cfg, epb, world, split):
    mesh = capi.Mesh(cfg())
    if mesh.ne < world:
        pytest.skip("fewer elements than partitions")
    for rank in range(world):
        h, roles = roles_of(mesh, world, rank, epb, split)
        nbr = h["nbr_local"]
        ne = nbr.shape[0]
        ghost_group = np.zeros((ne + epb - 1) // epb + 1, bool)
        for e in range(ne):
            if (nbr[e] <= -2).any():
                ghost_group[e // epb] = True
        for b in range(ne):
            for f in range(3):
                a = int(nbr[b, 2 * f])
                pulled = bool(roles[b] >> f & 1)
                if pulled:
                    # the pusher is a local element across that very face, dispatched no
                    # later than the puller, and it knows that it has to push
                    assert a >= 0 and a != b
                    assert int(nbr[a, 2 * f + 1]) == b
                    assert roles[a] >> (3 + f) & 1
                    if split:
                        # launch order: interior list first, then the boundary list
                        ka, kb = (ghost_group[a // epb], a), (ghost_group[b // epb], b)
                        assert ka < kb
                    else:
                        assert a < b
                else:
                    # evaluated by b itself: wall, ghost, wrap-around, self-neighbour, other list
                    if split and a >= 0:
                        later = (ghost_group[a // epb], a) >= (ghost_group[b // epb], b)
                    else:
                        later = a >= b
                    assert a < 0 or later or int(nbr[a, 2 * f + 1]) != b, (b, f, a)
            for d in range(3):
                if roles[b] >> (3 + d) & 1:
                    a = int(nbr[b, 2 * d + 1])
                    assert a != b and roles[a] >> d & 1 and int(nbr[a, 2 * d]) == b
        # pushes and pulls pair up one to one
        assert sum(bin(int(r) & 7).count("1") for r in roles) == sum(bin(int(r) >> 3).count("1") for r in roles)


def test_interior_elements_evaluate_three_faces():
    """On a periodic mesh cut nowhere, away from the wrap-around every element
    evaluates its three + faces and pulls its three - faces: the face work is
    halved."""
    mesh = capi.Mesh(capi.bubble_mesh_config(3, True))
    _, roles = roles_of(mesh, 1, 0, 5, False)
    pulls = np.array([bin(int(r) & 7).count("1") for r in roles])
    # 8^3 elements: a - face is pulled unless it wraps around (1/8 of them per direction)
    assert pulls.sum() == 3 * 512 - 3 * 64
    assert (pulls == 3).sum() == 7 ** 3
