"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): K2 ring step, K1 via the machine
(staged, direct and gather batches, events and completion words), K6 hydro
(ghosted and lattice/TMA, dynamic assignment), K7 FMM (one device and slab
geometry), star step and its slab decomposition, the hydro machine."""
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
    # round 2: direct batches (k_launch_gather_edge: fold + reductions) with
    # events and with completion words (the last CTA's counter and word),
    # gather batches with words, a batch wider than one launch, and K6 on
    # enough sub-grids for its dynamic work counter to hand out more
    for comp in ("events", "words"):
        run_native(16, 2, workers=2, executors=2, max_agg=4, mode=IntegrationMode.POLLING,
                   zero_copy=4, completion=comp)
    run_native(16, 1, workers=2, executors=2, max_agg=4, mode=IntegrationMode.FENCE,
               zero_copy=2, completion="words")
    run_native(64, 1, workers=2, executors=1, max_agg=300, mode=IntegrationMode.POLLING,
               zero_copy=4, completion="words")
    I3, dx3 = rotating_star(512, device=dev)
    hydro_flux(with_ghosts(I3), dx3)
    run_native_hydro(rotating_star(8)[0].numpy(), 1, workers=2, executors=2, max_agg=4)
    torch.cuda.synchronize()
    print("cases ok")


if __name__ == "__main__":
    main()
