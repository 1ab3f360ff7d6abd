"""Host-side logic of the drop-in package (CPU only): the master state
machine (mirrors reference tests/test_scheduler.py), PSF/volume generators
(bitwise the reference's draws, pinned by the golden kernels), slab support
known answers (reference tests/test_blur.py:122-137), configs, flop counts."""

import io

import numpy as np
import pytest

from conftest import golden
from paper_2002_02328_b200 import blur, configs, runtime, scheduler
from paper_2002_02328_b200.blur import KernelDims, dirac_stack
from paper_2002_02328_b200.scheduler import (ProtocolError, UpdateMessage, delay_stats, init_master, make_task,
                                             next_block, partition_blocks, receive_update, roll_sweep,
                                             should_stop, sweep_complete, write_trace_csv)
from paper_2002_02328_b200.volume import Dims3, SliceBlock, ellipsoid_phantom, init_uniform


def fresh(nz=24, workers=4, height=1, nx=3, ny=2):
    psf = dirac_stack(Dims3(nx, ny, nz), KernelDims(1, 1, 3))
    x0 = np.arange(nx * ny * nz, dtype=np.float64).reshape(nz, ny, nx) / 100.0
    return init_master(x0, workers, height, psf)


def answer(task, inc=None):
    return UpdateMessage(task.worker_id, task.block, np.zeros(task.d_mem.shape) if inc is None else inc, task.issue_k)


class TestScheduler:
    def test_partition_and_init(self):
        state, tasks = fresh(nz=24, workers=4)
        assert [t.block for t in tasks] == [SliceBlock(z, z) for z in range(4)]
        assert state.cursor == 4 and state.k == 0
        assert partition_blocks(7, 3) == [SliceBlock(0, 2), SliceBlock(3, 5), SliceBlock(6, 6)]
        with pytest.raises(ValueError, match="exceed"):
            fresh(nz=4, workers=3, height=2)

    def test_receive_update_locality_and_errors(self):
        state, tasks = fresh()
        before = state.x.copy()
        inc = np.zeros(6)
        inc[2] = 1.0
        receive_update(state, answer(tasks[1], inc))
        assert (state.x != before).sum() == 1 and state.k == 1
        with pytest.raises(ProtocolError, match="no in-flight"):
            receive_update(state, UpdateMessage(99, tasks[0].block, np.zeros(6), 0))
        with pytest.raises(ProtocolError, match="expected"):
            receive_update(state, UpdateMessage(1, SliceBlock(5, 5), np.zeros(6), 0))
        with pytest.raises(ProtocolError, match="non-finite"):
            receive_update(state, answer(tasks[0], np.full(6, np.nan)))
        with pytest.raises(ProtocolError, match="length"):
            receive_update(state, answer(tasks[0], np.zeros(5)))

    def test_single_worker_cycle_and_memory(self, rng):
        state, tasks = fresh(nz=5, workers=1)
        task, seq, stored = tasks[0], [tasks[0].block], {}
        for _ in range(9):
            inc = rng.standard_normal(task.d_mem.shape)
            if task.block in stored:
                assert np.array_equal(task.d_mem, stored[task.block])
            else:
                assert not task.d_mem.any()
            receive_update(state, answer(task, inc))
            stored[task.block] = inc
            task = make_task(state, 1, next_block(state, 1))
            seq.append(task.block)
        assert seq == [SliceBlock(z % 5, z % 5) for z in range(10)]

    def test_skip_rule_and_disjointness(self):
        state, tasks = fresh(nz=3, workers=2)
        receive_update(state, answer(tasks[0]))
        state.cursor = 1
        assert next_block(state, 1) == SliceBlock(2, 2)
        state, tasks = fresh(nz=6, workers=3)
        task = tasks[0]
        for _ in range(30):
            receive_update(state, answer(task))
            held = {a.block_index for a in state.in_flight.values()}
            blk = next_block(state, task.worker_id)
            assert state.blocks.index(blk) not in held
            task = make_task(state, task.worker_id, blk)

    def test_snapshot_and_support(self):
        state, tasks = fresh()
        t = tasks[0]
        assert t.slab == blur.slab_support(state.psf, t.block)
        state.x += 1.0
        assert not np.array_equal(t.x_slab, state.x[t.slab.z_lo:t.slab.z_hi + 1])

    def test_stop_rule(self, rng):
        state, tasks = fresh(nz=4, workers=1)
        task = tasks[0]
        while not sweep_complete(state):
            receive_update(state, answer(task))
            if sweep_complete(state):
                break
            task = make_task(state, 1, next_block(state, 1))
        assert should_stop(state, 1e-12)
        assert should_stop(state, np.inf)
        roll_sweep(state)
        assert not sweep_complete(state)
        assert should_stop(state, 1e-6, max_updates=4)
        assert should_stop(state, 1e-6, norms=(0.0, 1.0))
        assert not should_stop(state, 1e-6, norms=(1.0, 1.0))
        with pytest.raises(ValueError):
            should_stop(state, 0.0)

    def test_staleness_ledger_and_trace_csv(self):
        state, tasks = fresh(nz=9, workers=3)
        pending = {t.worker_id: t for t in tasks}
        for i in range(30):
            wid = (i % 3) + 1
            task = pending.pop(wid)
            receive_update(state, answer(task))
            pending[wid] = make_task(state, wid, next_block(state, wid))
        st, tau = delay_stats(state)
        assert tau <= 2 and max(st) == tau
        buf = io.StringIO()
        write_trace_csv(state.trace[:2], buf)
        lines = buf.getvalue().strip().splitlines()
        assert lines[0] == "event_index,worker_id,z_lo,z_hi,issue_k,receipt_k,staleness"
        assert lines[1].startswith("0,1,0,0,0,0,0")


class TestGenerators:
    def test_psf_stacks_bitwise_reference(self):
        """generate_psf_stack draws = the reference's (golden kernels were
        produced by the reference with the same seeds)."""
        specs = [((10, 9, 8), (5, 3, 5), 6), ((8, 8, 6), (3, 5, 3), 2), ((12, 8, 12), (3, 3, 3), 5)]
        g = golden("blur")
        for i, (dims, kd, seed) in enumerate(specs):
            psf = blur.generate_psf_stack(Dims3(*dims), KernelDims(*kd), seed=seed)
            assert np.array_equal(psf.kernels, g[f"blur{i}"]["kernels"])
            assert np.array_equal(psf.params, g[f"blur{i}"]["params"])

    def test_baseline_psf_family_bitwise_reference(self):
        cfg = configs.CONFIGS["C1"]
        psf = blur.depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
        assert np.array_equal(psf.kernels, golden("c1")["kernels"])

    def test_psf_validation(self):
        with pytest.raises(ValueError, match="odd"):
            KernelDims(2, 3, 3).validate()
        with pytest.raises(ValueError, match="positive"):
            blur.gaussian_kernel(KernelDims(3, 3, 3), 0.0, 1.0, 1.0, 0, 0)
        with pytest.raises(ValueError, match="exceeds"):
            blur.generate_psf_stack(Dims3(4, 4, 2), KernelDims(3, 3, 5), seed=0)
        with pytest.raises(ValueError, match="sum"):
            blur.PsfStack(Dims3(3, 3, 2), KernelDims(1, 1, 1), np.full((2, 1, 1, 1), 0.5))

    def test_slab_support_known_answers(self):
        assert blur.slab_support(dirac_stack(Dims3(4, 4, 8), KernelDims(1, 1, 1)), SliceBlock(3, 3)) == SliceBlock(2, 4)
        assert blur.slab_support(dirac_stack(Dims3(4, 4, 24), KernelDims(3, 3, 5)), SliceBlock(10, 10)) == SliceBlock(5, 15)
        assert blur.slab_support(dirac_stack(Dims3(4, 4, 8), KernelDims(3, 3, 5)), SliceBlock(0, 1)) == SliceBlock(0, 6)
        assert blur.slab_support(dirac_stack(Dims3(4, 4, 8), KernelDims(3, 3, 3)), SliceBlock(6, 7)) == SliceBlock(3, 7)

    def test_flops_formula(self):
        # nnz(H) = prod_i (n_i k_i - r_i(r_i+1)); C2: 2*nnz = 2.188 GFLOP
        assert blur.flops_H(Dims3(256, 256, 64), KernelDims(5, 5, 11)) == 2187906448
        assert blur.flops_H(Dims3(5, 4, 3), KernelDims(1, 1, 1)) == 2 * 60

    def test_ellipsoid_phantom(self):
        a = ellipsoid_phantom(Dims3(32, 24, 16), 10, 3)
        assert np.array_equal(a, ellipsoid_phantom(Dims3(32, 24, 16), 10, 3))
        assert a.min() >= 0 and a.max() > 0
        g = ellipsoid_phantom(Dims3(32, 24, 16), 10, 3, amplitude="gamma")
        assert g.max() > 0 and not np.array_equal(a, g)

    def test_init_uniform(self):
        x = init_uniform(Dims3(4, 3, 2), 2.0, 5)
        assert x.shape == (2, 3, 4) and x.min() >= 0 and x.max() <= 2.0
        assert not init_uniform(Dims3(4, 3, 2), 0.0, 5).any()

    def test_run_config_validation(self):
        with pytest.raises(ValueError):
            runtime.RunConfig(method="nope")
        with pytest.raises(ValueError):
            runtime.RunConfig(engine="nope")
        with pytest.raises(ValueError):
            runtime.RunConfig(workers=0)
        with pytest.raises(ValueError):
            runtime.RunConfig(tol=0.0)
        with pytest.raises(ValueError):
            runtime.RunConfig(dtype="f16")

    def test_configs_cover_baseline(self):
        assert set(configs.CONFIGS) >= {"C1", "C2", "C3", "C4", "C5"}
        c = configs.CONFIGS["C5"]
        assert c.dims == Dims3(1024, 1024, 512) and c.kdims == (9, 9, 21) and c.dtype == "f32"


def test_raise_step_status_maps_reference_errors():
    """StepInfo status column -> the reference's error at the same point:
    1 = non-finite gradient (ValueError from subspace_step,
    directions.py:64-65), 2 = non-finite increment (ProtocolError from
    receive_update, scheduler.py:147-148); the first failed step decides."""
    import pytest
    from paper_2002_02328_b200 import scheduler
    scheduler.raise_step_status(np.zeros(5))
    with pytest.raises(ValueError, match="non-finite gradient"):
        scheduler.raise_step_status(np.array([0.0, 1.0, 2.0]))
    with pytest.raises(scheduler.ProtocolError, match="non-finite increment"):
        scheduler.raise_step_status(np.array([0.0, 2.0, 1.0]))
