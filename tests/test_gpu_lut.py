"""K6: the paper's LUT GEMV (lutgemm.cpp:11-71) on the GPU -- a comparison
line, not the product path.  Its tables are bit-identical to the reference's
(same ascending-k float operations); its lookups are summed in a different
order, so it matches the C port's LUT gemv to ~1e-6 and the fp32 oracle
matmul_reference within the 1e-3 bar."""
import numpy as np
import pytest

from synth import activations, errors, model_bytes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,bits,mb,nb", [((4096, 4096), 3.5, 512, 128), ((1024, 2048), 2.5, 128, 256),
                                              ((512, 1024), 5.5, 64, 128)])
@pytest.mark.parametrize("M", [1, 3])
def test_lut_kernel_matches_reference_lut(gpu, port, shape, bits, mb, nb, M):
    import torch
    rows, cols = shape
    data = model_bytes(port, rows, cols, bits, m_b=mb, n_b=nb)
    dm = gpu.DeviceModel(data, flags=gpu.MODEL_LUT_LAYOUT)
    pm = port.load(data)
    x = activations(port, M, cols, seed=M + 40)
    y = dm.gemm(torch.from_numpy(x).cuda(), path=gpu.PATH_LUT).cpu().numpy()
    y_lut = np.stack([pm.gemv_lut(x[t])[0] for t in range(M)])
    assert errors(y, y_lut)[0] <= 1e-5
    assert errors(y, port.matmul(x, pm.dequantize(), threads=8))[0] <= 1e-3


def test_lut_path_requirements(gpu, port):
    import torch
    data = model_bytes(port, 1024, 1024, 3.25)
    plain = gpu.DeviceModel(data)
    x = torch.zeros(1, 1024, device="cuda")
    with pytest.raises(gpu.UnsupportedError):
        plain.gemm(x, path=gpu.PATH_LUT)
    lut = gpu.DeviceModel(data, flags=gpu.MODEL_LUT_LAYOUT)
    with pytest.raises(gpu.UnsupportedError):
        lut.gemm(x.to(torch.bfloat16), path=gpu.PATH_LUT)
