"""Small workload for compute-sanitizer (one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
Runs K1 over golden and random shapes (every plan variant family, the
i-chunked path, unaligned totals, z sub-ranges), K2, K3, K4-free LF5 path
and the projector kernels, each checked against the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from oracle.hprime_oracle import hprime_oracle
    from paper_2003_09133_b200 import hprime_device
    from paper_2003_09133_b200.synth import random_psf_like_reference
    from paper_2003_09133_b200.verify import compare_device, plane_sums_device

    def dev(H):
        return torch.from_numpy(np.array(H.reshape(-1, order="F"))).cuda().view(H.shape[::-1]).permute(4, 3, 2, 1, 0)

    def host(t):
        return t.permute(4, 3, 2, 1, 0).contiguous().cpu().numpy().reshape(-1)

    shapes = [((55, 55, 11, 11, 2), np.float32), ((27, 20, 13, 5, 2), np.float64), ((66, 41, 21, 9, 1), np.float32),
              ((5, 3, 3, 3, 1), np.float32), ((8, 12, 7, 3, 3), np.float32), ((1, 1, 1, 1, 3), np.float64)]
    envs = [{}, {"LFBP_STAGE_MAX_KB": "2"}, {"LFBP_STAGES": "1"}, {"LFBP_SUBWARP": "32", "LFBP_CONSUMER_WARPS": "3"},
            {"LFBP_STAGE_KB": "1", "LFBP_SUBWARP": "8"}, {"LFBP_KFLAGS": "32"},
            {"LFBP_KFLAGS": "160", "LFBP_CONSUMER_WARPS": "3"}, {"LFBP_KFLAGS": "200", "LFBP_ZCHUNK_MB": "1"}]
    n = 0
    for env in envs:
        for k in ("LFBP_STAGE_MAX_KB", "LFBP_STAGES", "LFBP_SUBWARP", "LFBP_CONSUMER_WARPS", "LFBP_STAGE_KB",
                  "LFBP_KFLAGS", "LFBP_ZCHUNK_MB"):
            os.environ.pop(k, None)
        os.environ.update(env)
        for shape, dt in shapes:
            H = random_psf_like_reference(shape, density=0.9, seed=3, dtype=dt)
            out = hprime_device(dev(H))
            torch.cuda.synchronize()
            assert host(out).tobytes() == hprime_oracle(H).tobytes(order="F"), (env, shape)
            n += 1
    H = random_psf_like_reference((21, 19, 7, 5, 6), density=1.0, seed=3, dtype=np.float32)
    src = dev(H)
    out = torch.zeros_like(src)
    hprime_device(src, out=out, z_range=(2, 5))
    assert compare_device(out, out) == (0, -1)
    plane_sums_device(src, H.shape)
    from paper_2003_09133_b200 import Dims5, PsfArray, compute_backprojection
    from paper_2003_09133_b200.arrays import Image, Volume
    from paper_2003_09133_b200.projector import backproject, forward_project
    psf = PsfArray._wrap(Dims5(9, 9, 3, 3, 2), random_psf_like_reference((9, 9, 3, 3, 2), density=0.5, seed=1))
    bp = compute_backprojection(psf)
    forward_project(psf, Volume(np.ones((13, 11, 2))))
    backproject(bp, Image(np.ones((13, 11))))
    torch.cuda.synchronize()
    print(f"sanitize probe ok: {n} K1 launches checked")


if __name__ == "__main__":
    main()
