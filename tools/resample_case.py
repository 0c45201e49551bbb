import sys; sys.path.insert(0, '.')
import torch, paper_2203_10213_b200 as vk
v = vk.synthetic_device((512, 512, 512), vk.DataFormat.UINT8, seed=7)
for _ in range(3):
    vk.resample(v, (256, 256, 256))
torch.cuda.synchronize()
