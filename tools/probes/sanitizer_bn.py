import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1910_00078_b200.primkit import library
import test_bn_device_gpu as t
lib = library()
for shape in [(8, 64, 28), (4, 2048, 7)]:
    for relu in (0, 1):
        t._run(lib, *shape, relu, seed=1)
print("bn sanitizer run ok")
