"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): K2 ring step, K1 via the machine, K6
hydro (ghosted and lattice/TMA), K7 FMM (one device and slab geometry),
star step and its slab decomposition, the hydro machine."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2303_08058_b200 import _native as N
    from paper_2303_08058_b200.bridge import IntegrationMode
    from paper_2303_08058_b200.gravity import GravitySolver, rotating_star_density
    from paper_2303_08058_b200.hydro import hydro_flux, rotating_star, with_ghosts
    from paper_2303_08058_b200.native_machine import run_native, run_native_hydro
    from paper_2303_08058_b200.ring import RingStepper
    from paper_2303_08058_b200.star import RotatingStarStep
    from paper_2303_08058_b200.star_dist import VirtualCluster
    dev = torch.device("cuda", 0)
    N.init(0)
    st = RingStepper(64, device=dev, max_steps=4)
    st.step()
    st.step()
    I, dx = rotating_star(8, device=dev)
    hydro_flux(with_ghosts(I), dx)
    g = GravitySolver(2, dev)
    g.solve(rotating_star_density(2, device=dev))
    s1 = RotatingStarStep(2, device=dev)
    s1.step()
    vc = VirtualCluster(2, 2, s1.U.clone())
    vc.step()
    run_native(16, 1, workers=2, executors=2, max_agg=4, mode=IntegrationMode.POLLING)
    run_native_hydro(rotating_star(8)[0].numpy(), 1, workers=2, executors=2, max_agg=4)
    torch.cuda.synchronize()
    print("cases ok")


if __name__ == "__main__":
    main()
