import time, numpy as np, os
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip(), '|', open('/sys/kernel/mm/transparent_hugepage/defrag').read().strip())
for rep in range(3):
    t0 = time.perf_counter(); a = np.zeros((1 << 20, 128), np.float32); t1 = time.perf_counter()
    a[:] = 1.0; t2 = time.perf_counter()
    a[:] = 2.0; t3 = time.perf_counter()
    print(f'alloc {t1-t0:.4f} first touch {t2-t1:.4f} second write {t3-t2:.4f}')
    del a
a = np.empty((1 << 20, 128), np.float32)
t1 = time.perf_counter(); a[:] = 1.0; t2 = time.perf_counter()
print(f'np.empty first touch {t2-t1:.4f}')
