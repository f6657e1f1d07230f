"""Does this box expose NVLink SHARP (NVLS) / multicast?  NCCL's init log + the
driver attribute CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED."""
import ctypes, os, torch, torch.distributed as dist
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
t = torch.ones(1 << 26, device="cuda")
dist.all_reduce(t)
torch.cuda.synchronize()
cuda = ctypes.CDLL("libcuda.so.1")
v = ctypes.c_int(-1)
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
r = cuda.cuDeviceGetAttribute(ctypes.byref(v), CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, local)
if rank == 0:
    print("multicast_supported", r, v.value, flush=True)
dist.destroy_process_group()
