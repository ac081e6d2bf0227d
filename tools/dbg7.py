import sys; sys.path.insert(0,'.')
import numpy as np, paper_1306_5390_b200 as P
img = P.GrayImage(7,7,100); img.set(3,3,255); img.set(3,4,255)
for k in (1,2):
    r = P.denoise(img, P.DenoiseParams(max_iterations=k))
    print(k, [(s.flagged,s.replaced) for s in r.stats]); print(r.image.pixels)
